#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
nvidia-smi topo -m 2>&1 | head -8
lscpu | grep -i "numa\|socket\|model name"
python scripts/pcie_probe.py none
python scripts/pcie_probe.py local
