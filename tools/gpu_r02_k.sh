# Round 2, call K: progressive token-row epilogue stores; fold A/B at large T.
export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_gpu_linear_smoke.py tests/test_gpu_kernels.py tests/test_gpu_conv_igemm.py tests/test_gpu_fold.py -q -p no:cacheprovider > gpurun_out/r02k_pytest.log 2>&1
tail -4 gpurun_out/r02k_pytest.log
timeout 300 python tools/bench_linear.py --only bert_b8_qkv,bert_b8_proj_res,bert_b8_ff1_gelu,bert_b8_ff1,bert_b8_ff2_res,xlnet_b4_ff1_gelu > gpurun_out/r02k_linear.jsonl 2>&1
cut -c1-150 gpurun_out/r02k_linear.jsonl
for C in C5 C4; do timeout 600 python tools/ab_plan.py --config $C --variants fold_ln=1 fold_ln=0 2>&1 | tail -3; done
timeout 600 python tools/ab_plan.py --config C3 --variants fuse=1 2>&1 | tail -1
