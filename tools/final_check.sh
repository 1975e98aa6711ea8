timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['metric'], d['value']/1e9, 'G', 'frac', d['roofline']['frac'], 'l2', d['roofline']['l2_request_roofline']['frac'], 'e2e', d['e2e']['value']/1e9, 'cpu', d['cpu_baseline']['value']/1e6, 'M', d['clocks'], d['gpu_launches'])"
timeout 900 python bench.py --impl reference 2>/dev/null | tail -1 | cut -c1-200
