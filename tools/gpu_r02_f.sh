# Round 2, call F: epilogue TMEM prefetch + fp32 GEMV heads + TF32 split cap.
export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_linear_smoke.py tests/test_gpu_fold.py tests/test_gpu_conv_tf32.py tests/test_gpu_conv_igemm.py -q -x -p no:cacheprovider > gpurun_out/r02f_pytest.log 2>&1
tail -3 gpurun_out/r02f_pytest.log
timeout 300 python tools/bench_linear.py --only bert_b8_qkv,bert_b8_proj_res,bert_b8_ff1_gelu,bert_b8_ff2_res,bert_b8_ff1,bert_b8_ff2,xlnet_b4_ff1_gelu > gpurun_out/r02f_linear.jsonl 2>&1
cat gpurun_out/r02f_linear.jsonl | cut -c1-200
for C in C5 C1; do
timeout 600 python bench.py --config $C --no-unmerged --no-cpu > gpurun_out/r02f_bench_$C.log 2>&1; tail -1 gpurun_out/r02f_bench_$C.log | cut -c1-330
done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider > gpurun_out/r02f_configs.log 2>&1; tail -2 gpurun_out/r02f_configs.log
