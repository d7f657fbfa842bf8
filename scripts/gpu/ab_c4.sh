cd "${GRAFT_REPO_ROOT:-/root/repo}"
for n in "$@"; do
  L=paper_1802_06215_b200/libdespot_$n.so; [ "$n" = base ] && L=paper_1802_06215_b200/libdespot.so
  DESPOT_LIB=$L timeout 300 python bench.py --config 4 --no-cpu-baseline --no-all-cores-baseline > gpurun_out/ab_$n.json 2>&1
  tail -1 gpurun_out/ab_$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$n\", round(d[\"ms_per_step\"],4), round(d[\"phases_ms\"][\"K2_expand_rollout\"],4))" || tail -3 gpurun_out/ab_$n.json
done
