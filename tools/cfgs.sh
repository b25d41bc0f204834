cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in C3 C4 C5; do
  timeout 1200 python tools/run_config.py $c --sample 96 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
done
