#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py -q -p no:cacheprovider --timeout 300 -rf -k "tile5 or edge_shapes or chunking" > gpurun_out/pytest_t40.txt 2>&1
tail -2 gpurun_out/pytest_t40.txt
for at in 1 0; do for c in c2 c3 c4 c5 c2f64 c5f64; do
  r=$(TF_TILE_AUTOTUNE=$at timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-simp --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), round(d.get('warm_l2_ms_per_step',0)*1e3,2))")
  echo "autotune=$at $c: GDOF/s us(flushed) us(warm) = $r"
done; done
