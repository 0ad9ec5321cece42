#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 1800 python -m pytest tests -q -p no:cacheprovider --timeout 900 -m gpu 2>&1 | grep -E "^E |passed|failed|Error|FAILED" | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench91.json 2> gpurun_out/bench91.err
tail -c 400 gpurun_out/bench91.err
python -c "
import json; d=json.loads(open('gpurun_out/bench91.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ['value','ms_per_step','e2e','clocks','gpu_launches']})
print('roof', d['roofline']['frac'], d['roofline']['fma']['frac'], 'cpu', d['cpu_baseline']['value'] if d['cpu_baseline'] else None)
print('simp', d['simp']['s_per_iter'], 'simp_c2', d['simp_c2']['s_per_iter'], d['simp_c2']['wall_s'], 'c4', d['simp_c4_scaling']['s_per_iter'])
print('cg', d['cg'])
"
