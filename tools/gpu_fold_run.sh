export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_linear_smoke.py tests/test_gpu_fold.py -q --timeout 300 2>&1 | tail -1
for i in 1 2; do
echo "def $(timeout 300 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
echo "B32 $(timeout 300 python bench.py --no-unmerged --no-cpu --instances 32 2>&1 | tail -1 | cut -c150-210)"
done
