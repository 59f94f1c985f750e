export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_execute.py -q --timeout 300 -k pipelined 2>&1 | grep -E "Error|assert|passed|failed" | head -20
for i in 1 2; do timeout 300 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'])"; done
