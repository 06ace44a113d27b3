set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
PBNG_TRACE=1 timeout 200 python scripts/quick_run.py 4 --opts 8 --reps 1 > gpurun_out/r6_trace4.log 2>&1
PBNG_TRACE=1 timeout 400 python scripts/quick_run.py 5 --opts 8 --reps 1 > gpurun_out/r6_trace5.log 2>&1
timeout 200 python scripts/quick_run.py 4 --reps 1 > gpurun_out/r6_plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg_win -s 40 -c 3 -o gpurun_out/r6_prof_win4 python scripts/quick_run.py 4 --reps 1 > gpurun_out/r6_ncu.log 2>&1
echo "ncu rc=$?"
