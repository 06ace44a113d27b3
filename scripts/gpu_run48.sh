set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
export PBNG_CACHE=/tmp/pbng_graph_cache_r1
for c in 4 5; do
  for v in main noid; do
    lib=paper_2110_12511_b200/libpbng_$v.so; [ $v = main ] && lib=paper_2110_12511_b200/libpbng.so
    PBNG_LIB=$lib timeout 400 python scripts/quick_run.py $c --opts 8 --reps 2 2>&1 | grep '"rep"' > gpurun_out/r48_${v}_$c.log
  done
done
for f in gpurun_out/r48_*_?.log; do echo $f; tail -1 $f | cut -c1-160; done
timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/r48_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r48_pytest.log
