import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2009_13062_b200 import _lib
torch.manual_seed(0)
st = torch.cuda.current_stream().cuda_stream
for T in (128, 200, 256):
  for K, N in ((64, 64), (256, 64)):
    for use_bias, act in ((False, 0), (True, 0), (False, 1), (True, 1)):
        x = (torch.rand(1, T, K, device='cuda') - .5).bfloat16()
        w = (torch.rand(1, N, K, device='cuda') - .5).bfloat16()
        b = (torch.rand(1, N, device='cuda') - .5).float()
        r = (torch.rand(1, T, N, device='cuda') - .5).bfloat16()
        y = torch.empty(1, T, N, device='cuda', dtype=torch.bfloat16)
        for res in (None, r):
            _lib.call("nf_grouped_linear_ws", x.data_ptr(), K, T*K, w.data_ptr(), b.data_ptr() if use_bias else None,
                      res.data_ptr() if res is not None else None, y.data_ptr(), N, T*N, 1, T, K, N, 1, 0, act, 0, None, 0, st)
            torch.cuda.synchronize()
            ref = x.float()[0] @ w.float()[0].T
            if use_bias: ref = ref + b[0]
            if res is not None: ref = ref + r.float()[0]
            if act: ref = torch.relu(ref)
            err = ((y.float()[0] - ref).abs().max() / ref.abs().max()).item()
            if err > 1e-2: print("BAD", T, K, N, use_bias, act, res is not None, err)
print("done")
