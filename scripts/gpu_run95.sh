#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
start=$(date +%s)
timeout 2400 python -m pytest tests -q -p no:cacheprovider --timeout 900 -m gpu 2>&1 | grep -E "^E |passed|failed|Error|FAILED" | head -20
echo "gpu suite seconds: $(( $(date +%s) - start ))"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench95.json 2> gpurun_out/bench95.err
tail -c 300 gpurun_out/bench95.err
python -c "
import json; d=json.loads(open('gpurun_out/bench95.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ['value','ms_per_step','e2e','clocks','gpu_launches']})
print('simp', d['simp']['s_per_iter'], 'simp_c2', d['simp_c2']['s_per_iter'], d['simp_c2']['wall_s'], 'c4', d['simp_c4_scaling']['s_per_iter'])
print('cg', {k: (v.get('protocol'), v.get('us_per_iteration')) for k, v in d['cg'].items() if k in ('fp32','fp64')})
"
