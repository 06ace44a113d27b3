set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
export PBNG_CACHE=/tmp/pbng_graph_cache_r1 PBNG_TRACE=1
timeout 600 python scripts/quick_run.py 5 --reps 1 > gpurun_out/r43_plain5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_agg_win -s 60 -c 1 -o gpurun_out/r43_prof_win5 python scripts/quick_run.py 5 --reps 1 > gpurun_out/r43_ncu.log 2>&1
echo "ncu rc=$?"
