set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "not config4 and not config5" > gpurun_out/r42_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r42_pytest.log
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
for v in main; do
  lib=paper_2110_12511_b200/libpbng_$v.so; [ $v = main ] && lib=paper_2110_12511_b200/libpbng.so
  for c in 3 4 5; do
    PBNG_LIB=$lib timeout 400 python scripts/quick_run.py $c --opts 8 --reps 2 2>&1 | grep -v "^cd \|^fd part" > gpurun_out/r42_${v}_$c.log
  done
done
for f in gpurun_out/r42_*_?.log; do echo $f; grep -h "rep" $f | tail -1 | cut -c1-200; done
