# Round 2, call H: token-row folded LayerNorm (large T) + 192-wide tiles gate.
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_linear_smoke.py -q -x -p no:cacheprovider > gpurun_out/r02h_pytest.log 2>&1
tail -3 gpurun_out/r02h_pytest.log
for C in C5 C4; do
timeout 600 python bench.py --config $C --no-unmerged --no-cpu > gpurun_out/r02h_bench_$C.log 2>&1; tail -1 gpurun_out/r02h_bench_$C.log | cut -c1-330
done
NF_PARITY_LOG=gpurun_out/r02h_parity.jsonl timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_execute.py -q -x -p no:cacheprovider > gpurun_out/r02h_configs.log 2>&1; tail -3 gpurun_out/r02h_configs.log
