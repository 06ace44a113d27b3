set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in c00 c01 c11; do
  for c in 3 4 5; do
    PBNG_LIB=paper_2110_12511_b200/libpbng_$v.so timeout 300 python scripts/quick_run.py $c --opts 8 --reps $([ $c = 5 ] && echo 1 || echo 2) 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $c, round(d['ms'],1), round(d['ms_count'],1), round(d['ms_cd'],1), round(d['ms_fd'],1), d['ms_kernel'].get('agg_cta'), d['impl'])" >> gpurun_out/r21_sweep.txt
  done
done
cat gpurun_out/r21_sweep.txt
