# Round 2, call G: 192-wide CTA-pair tiles.
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_linear_smoke.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/r02g_pytest.log 2>&1
tail -3 gpurun_out/r02g_pytest.log
timeout 300 python tools/bench_linear.py --only bert_b8_proj_res,bert_b8_ff2_res,bert_b8_ff2,xlnet_b4_proj_res,xlnet_b4_ff2 > gpurun_out/r02g_linear.jsonl 2>&1
cat gpurun_out/r02g_linear.jsonl | cut -c1-200
timeout 600 python bench.py --config C5 --no-unmerged --no-cpu > gpurun_out/r02g_bench_C5.log 2>&1; tail -1 gpurun_out/r02g_bench_C5.log | cut -c1-330
timeout 600 python bench.py --config C4 --no-unmerged --no-cpu > gpurun_out/r02g_bench_C4.log 2>&1; tail -1 gpurun_out/r02g_bench_C4.log | cut -c1-330
