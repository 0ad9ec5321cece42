#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 600 python -c "
import bench, json
out = bench.kernel_sweep()
for k, v in out.items(): print(k, round(v['ms_per_step']*1e3, 1), 'us', round(v['GDOF_s'], 2), 'GDOF/s', round(v['hbm_frac'], 3))
"
