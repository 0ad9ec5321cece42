#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
TF_BENCH_SAME_DEVICE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu > gpurun_out/bench87_n2.json 2> gpurun_out/bench87_n2.err
tail -c 800 gpurun_out/bench87_n2.err | grep -v "OMP\|\*\*\*"
python -c "
import json; d=json.loads(open('gpurun_out/bench87_n2.json').read().strip().splitlines()[-1])
s = d['simp_c4_scaling']; print(s['path'], s['s_per_iter'], s['cg_iterations']); p = s.get('peer'); print(p.get('path'), p.get('s_per_iter'), p.get('error'))
"
