# Round 2, call B: the full GPU suite on the pruned library, sanitizer
# re-run, headline bench lines (C5 default, C2) for regression checks.
export PYTHONPATH=.
NF_PARITY_LOG=gpurun_out/r02b_parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  > gpurun_out/r02b_pytest.log 2>&1
tail -5 gpurun_out/r02b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; tail -2 gpurun_out/r02b_smoke.log
timeout 600 python bench.py --model bert-base --instances 8 --batch 1 --steps 30 --warmup 5 --no-unmerged --no-cpu \
  > gpurun_out/r02b_bench_c2.log 2>&1; tail -1 gpurun_out/r02b_bench_c2.log | cut -c1-400
timeout 600 python bench.py --model bert-base --instances 32 --batch 8 --steps 20 --warmup 5 --no-unmerged --no-cpu \
  > gpurun_out/r02b_bench_c5.log 2>&1; tail -1 gpurun_out/r02b_bench_c5.log | cut -c1-400
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_linear_smoke.py tests/test_gpu_conv_igemm.py tests/test_gpu_fold.py -q -p no:cacheprovider \
    > gpurun_out/r02b_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02b_sanitizer_$tool.log
done
