#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_host.py -q -p no:cacheprovider --timeout 300 -rf -k "tile5 or chunking or symbols or abi" > gpurun_out/pytest_t43.txt 2>&1
tail -2 gpurun_out/pytest_t43.txt
for i in 1 2; do for c in c2 c3 c4 c5 c2f64; do
  r=$(timeout 300 python bench.py --config $c --steps 300 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), round(d.get('warm_l2_ms_per_step',0)*1e3,2), d['config'].get('launch'))")
  echo "$c: GDOF/s us(flushed) us(warm) = $r"
done; done
