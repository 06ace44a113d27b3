set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in dc512 dc512nt dc1024 dc2048 dc1024nt; do
  for c in 4 5; do
    PBNG_TRACE=1 PBNG_LIB=paper_2110_12511_b200/libpbng_$v.so timeout 300 python scripts/quick_run.py $c --opts 8 --reps $([ $c = 5 ] && echo 1 || echo 2) 2>&1 | grep -v "^cd \|^fd " > gpurun_out/r26_${v}_$c.log
  done
done
for f in gpurun_out/r26_*.log; do echo $f; grep -h "tier2" $f | tail -1 | cut -c1-250; grep -h "rep" $f | tail -1 | cut -c1-200; done
