#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 300 python -c "
from paper_2604_18020_b200 import SimpConfig, default_schedule, make_preset, run_simp
for n in (4,5,6):
    try:
        r = run_simp(make_preset('cantilever', 0.2), SimpConfig(schedule=default_schedule(n)))
        print(n, 'ok', [round(h.compliance,4) for h in r.history])
    except Exception as e:
        print(n, 'fail', e)
" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_slab_simp.py tests/test_gpu_operator.py -q -p no:cacheprovider --timeout 600 -m gpu 2>&1 | grep -E "^E |passed|failed|Error" | head -30
PROBE_OUT=gpurun_out/probe_mbb32.npz timeout 300 python scripts/slab_simp_probe.py 2 mbb 8 fp32 2>&1 | tail -1
