cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in 1 3 2; do for r in 1 2; do for L in old new; do
  LIB=paper_1802_06215_b200/libdespot.so; [ $L = old ] && LIB=paper_1802_06215_b200/libdespot_old.so
  DESPOT_LIB=$LIB timeout 300 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline --no-all-cores-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$L', round(d['ms_per_step'],4), 'e2e %.4g' % d['e2e']['value'])"
done; done; done
