export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_fold.py tests/test_gpu_execute.py -q --timeout 300 2>&1 | tail -2
NF_FOLD_LN=1 timeout 300 python tools/profile_plan.py --no-pdl 2>&1 | grep -v Warn | head -5
for i in 1 2; do for f in 1 0; do
echo "fold=$f $(NF_FOLD_LN=$f timeout 300 python bench.py --no-cpu --no-unmerged 2>&1 | tail -1 | cut -c1-200)"
done; done
