#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 900 python bench.py --steps 200 --warmup 5 > gpurun_out/bench79.json 2> gpurun_out/bench79.err
tail -c 600 gpurun_out/bench79.err
python -c "
import json; d=json.loads(open('gpurun_out/bench79.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'], d['simp_c4_scaling'])
print(d['simp_c2']['s_per_iter'], d['simp']) 
"
TF_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu > gpurun_out/bench79_n2.json 2> gpurun_out/bench79_n2.err
tail -c 1500 gpurun_out/bench79_n2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench79_n2.json').read().strip().splitlines()[-1])
print(d['value'], d['simp_c4_scaling'])
"
