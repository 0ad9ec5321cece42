#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ./scripts/exchange_bench 2 256 2000 > gpurun_out/xchg26.txt 2>&1
cat gpurun_out/xchg26.txt
