#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
start=$(date +%s)
timeout 2400 python -m pytest tests -q -p no:cacheprovider --timeout 900 -m gpu 2>&1 | grep -E "^E |passed|failed|Error|FAILED" | head -20
echo "gpu suite seconds: $(( $(date +%s) - start ))"
TF_BENCH_SAME_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-cpu > gpurun_out/bench99_n2.json 2> gpurun_out/bench99_n2.err
tail -c 300 gpurun_out/bench99_n2.err | grep -v "OMP\|\*\*\*"
python -c "
import json; d=json.loads(open('gpurun_out/bench99_n2.json').read().strip().splitlines()[-1])
s = d['simp_c4_scaling']; print(d['value'], d['slab_transports']); print(s['path'], s['s_per_iter'], s['median_iter_s_after_first']); p = s.get('peer'); print(p.get('path'), p.get('s_per_iter'), p.get('error'))
"
