export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_fold.py tests/test_gpu_kernels.py tests/test_gpu_execute.py -q --timeout 300 -x 2>&1 | tail -3
for i in 1 2; do
echo "def $(timeout 120 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
done
timeout 300 python tools/profile_plan.py --no-pdl 2>&1 | grep -v -i warn | head -5
