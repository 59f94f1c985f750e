export PYTHONPATH=.
NF_SMALLT_NORMAL=1 timeout 300 python -m pytest tests/test_gpu_linear_smoke.py -q --timeout 300 2>&1 | tail -1
for i in 1 2; do for n in 0 1; do
echo "normal=$n $(NF_FOLD_LN=0 NF_SMALLT_NORMAL=$n timeout 300 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
echo "normal=$n B32 $(NF_FOLD_LN=0 NF_SMALLT_NORMAL=$n timeout 300 python bench.py --no-unmerged --no-cpu --instances 32 2>&1 | tail -1 | cut -c150-210)"
done; done
NF_FOLD_LN=0 NF_SMALLT_NORMAL=1 timeout 300 python tools/profile_plan.py --no-pdl 2>&1 | grep -v Warn | head -6
NF_FOLD_LN=0 NF_SMALLT_NORMAL=1 timeout 300 python tools/profile_plan.py 2>&1 | grep -v Warn | head -2; python tools/timeline_ends.py
