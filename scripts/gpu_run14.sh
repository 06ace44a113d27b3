set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python scripts/quick_run.py 5 --reps 1 > gpurun_out/r14_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg_win -s 45 -c 1 -o gpurun_out/r14_prof_win5 python scripts/quick_run.py 5 --reps 1 > gpurun_out/r14_ncu.log 2>&1
echo "ncu rc=$?"
