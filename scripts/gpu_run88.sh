#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
timeout 900 python -m pytest tests/test_slab.py -q -p no:cacheprovider --timeout 600 -m gpu -k peer 2>&1 | grep -E "^E |passed|failed|Error" | head -20
TF_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu --no-simp > gpurun_out/bench88_n2.json 2> gpurun_out/bench88_n2.err
tail -c 600 gpurun_out/bench88_n2.err | grep -v "OMP\|\*\*\*"
python -c "
import json; d=json.loads(open('gpurun_out/bench88_n2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['config']['workload'], d['slab_transports'])
"
