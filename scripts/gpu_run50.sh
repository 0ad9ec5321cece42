#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export PYTHONPATH="$GRAFT_REPO_ROOT:$PYTHONPATH"
echo "box env PYTORCH_CUDA_ALLOC_CONF=$PYTORCH_CUDA_ALLOC_CONF"
env | grep -i "cuda\|nccl\|torch" | head
python scripts/pcie_probe.py tf
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False python scripts/pcie_probe.py tf
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python scripts/pcie_probe.py tf
