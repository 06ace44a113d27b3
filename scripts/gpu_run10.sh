set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in c128 c256 cad c128d1 c128d1nt c512; do
  for c in 3 4; do
    PBNG_LIB=paper_2110_12511_b200/libpbng_$v.so timeout 120 python scripts/quick_run.py $c --opts 8 --reps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $c, round(d['ms'],1), round(d['ms_count'],1), round(d['ms_cd'],1), d['ms_kernel'].get('agg_cta'))" >> gpurun_out/r10_sweep.txt
  done
done
cat gpurun_out/r10_sweep.txt
