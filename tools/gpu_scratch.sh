# scratch A/B script rewritten per experiment (see DESIGN §5 for the measured knobs)
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_execute.py tests/test_gpu_linear_smoke.py -q --timeout 300 2>&1 | tail -1
for i in 1 2; do for t in 16 0; do
echo "tiny=$t $(NF_SPLITK_TINY_T=$t timeout 300 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | cut -c150-210)"
done; done
timeout 300 python tools/profile_plan.py --no-pdl 2>&1 | grep -v Warn | head -8
