#!/bin/bash
# One parameterised GPU-box runner (replaces the per-run scratch wrappers).
#   gpurun --timeout 1200 -- 'bash scripts/gpu.sh tests'        # pytest -m gpu
#   gpurun --timeout 900  -- 'bash scripts/gpu.sh bench'        # bench.py line
#   gpurun --timeout 900  -- 'bash scripts/gpu.sh launches'     # ncu launch list of the bench
#   gpurun --timeout 900  -- 'bash scripts/gpu.sh ncu KERNEL_REGEX -- python script.py args'
# Everything lands in gpurun_out/ (merged back by gpurun).
set -u
mkdir -p gpurun_out
what=${1:-tests}; shift || true
case "$what" in
  tests)
    timeout 2400 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/tests.log 2>&1
    echo "pytest exit $?"; tail -5 gpurun_out/tests.log ;;
  bench)
    timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
    echo "bench exit $?"; tail -c 3000 gpurun_out/bench.json ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 "$@" > gpurun_out/launches.log 2>&1
    echo "ncu exit $?" ;;
  ncu)
    k=$1; shift; [ "${1:-}" = "--" ] && shift
    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
      -o gpurun_out/ncu_full -f "$@" > gpurun_out/ncu.log 2>&1
    echo "ncu exit $?"; tail -3 gpurun_out/ncu.log ;;
  *) echo "unknown: $what"; exit 2 ;;
esac
