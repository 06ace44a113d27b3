set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "not config4 and not config5" > gpurun_out/r22_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r22_pytest.log
for v in pre32k pre1k; do
  for c in 4 5; do
    PBNG_TRACE=1 PBNG_LIB=paper_2110_12511_b200/libpbng_$v.so timeout 300 python scripts/quick_run.py $c --opts 8 --reps 1 2>&1 | grep -v "^cd \|^fd " > gpurun_out/r22_${v}_$c.log
  done
done
grep -h "tier2\|rep" gpurun_out/r22_pre*.log | cut -c1-330
