export PYTHONPATH=.
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'] if d.get('cpu_baseline') else None)"
