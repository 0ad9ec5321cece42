set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/tests_full.log 2>&1; echo pytest $?; tail -5 gpurun_out/tests_full.log
