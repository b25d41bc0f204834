#!/bin/bash
# tools/gpu_i.sh <tag> : all GPU tests, quick benches, ncu --set full of l2p / p2m at C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash tools/gpu_f.sh $1 C5 C2 C3 C4
bash tools/gpu_ncu.sh $1 "C5:l2p_kernel:1" "C5:p2m_kernel:1"
