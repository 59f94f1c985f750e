import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2009_13062_b200 import _lib, kernels as K
from oracle import kernels as OK
torch.manual_seed(0)
def nw(a,b): return float(np.max(np.abs(a-b))/np.max(np.abs(b)))
lib=_lib.load()
for (G, cg, coutg, H, k, s, p) in [(1, 64, 64, 16, 1, 1, 0), (1, 64, 64, 12, 1, 1, 0), (1, 128, 64, 16, 1, 1, 0), (1, 64, 128, 16, 1, 1, 0), (1, 64, 64, 11, 1, 1, 0), (2, 64, 64, 16, 3, 1, 1)]:
    C, Cout = G*cg, G*coutg
    x = OK.bf16_round(np.random.uniform(-1,1,(1,C,H,H)).astype(np.float32))
    w = OK.bf16_round(np.random.uniform(-.2,.2,(Cout,cg,k,k)).astype(np.float32))
    want = OK.grouped_conv2d(x, w, groups=G, stride=s, padding=p)
    xn = torch.from_numpy(x).cuda().bfloat16().permute(0,2,3,1).contiguous()
    Ho = (H+2*p-k)//s+1
    pix = Ho*Ho
    kk = k*k*cg; kpad = -(-kk//8)*8
    wf = torch.from_numpy(w).cuda().permute(0,2,3,1).reshape(G, coutg, kk)
    wf = torch.nn.functional.pad(wf, (0, kpad-kk)).bfloat16().contiguous()
    y = torch.empty(1, Ho, Ho, Cout, device='cuda', dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    if k == 1:
        xp, xld, xgs, kd = xn.data_ptr(), C, cg, cg
    else:
        col = torch.empty(pix, G, kpad, device='cuda', dtype=torch.bfloat16)
        _lib.call("nf_im2col_nhwc", xn.data_ptr(), col.data_ptr(), 1, H, H, C, G, k, s, p, kpad, 1, st)
        xp, xld, xgs, kd = col.data_ptr(), G*kpad, kpad, kpad
        # check im2col vs torch unfold
    _lib.call("nf_grouped_linear_ws", xp, xld, xgs, wf.data_ptr(), None, None, y.data_ptr(), Cout, coutg, G, pix, kd, coutg, 1, 0, 0, 0, None, 0, st)
    torch.cuda.synchronize()
    got = y.permute(0,3,1,2).float().cpu().numpy()
    print((G,cg,coutg,H,k,s,p), "err", nw(got, want))
    # dense GEMM reference for the 1x1 case through strided API with G=1 per group
    if k == 1 and G > 1:
        for g in range(G):
            sub = got[:, g*coutg:(g+1)*coutg]; wsub = want[:, g*coutg:(g+1)*coutg]
            print("  group", g, nw(sub, wsub))
