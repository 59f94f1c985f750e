export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_fold.py tests/test_gpu_linear_smoke.py tests/test_gpu_execute.py -q --timeout 300 -x 2>&1 | tail -2
for i in 1 2 3; do
echo "new $(timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
done
