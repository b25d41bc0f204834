cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/p2p_var.jsonl
for c in C1x C2 C3 C4; do timeout 300 python tools/phase_bench.py $c --reps 3 >> gpurun_out/p2p_var.jsonl 2>>gpurun_out/p2p_var.err; done
