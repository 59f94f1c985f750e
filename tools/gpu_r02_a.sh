# Round 2, first GPU call: BASELINE-config parity through the bench plan,
# compute-sanitizer over the kernel unit tests, the new default bench line.
export PYTHONPATH=.
nproc > gpurun_out/r02a_nproc.txt
NF_PARITY_LOG=gpurun_out/r02a_parity.jsonl timeout 1500 python -m pytest tests/test_gpu_configs.py -v -s \
  > gpurun_out/r02a_configs.log 2>&1
tail -15 gpurun_out/r02a_configs.log
timeout 600 python bench.py --model bert-base --instances 32 --batch 8 --steps 20 --warmup 5 --no-unmerged \
  > gpurun_out/r02a_bench_c5.log 2>&1; tail -1 gpurun_out/r02a_bench_c5.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_linear_smoke.py tests/test_gpu_conv_igemm.py tests/test_gpu_fold.py -x -q -p no:cacheprovider \
    > gpurun_out/r02a_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r02a_sanitizer_$tool.log
done
