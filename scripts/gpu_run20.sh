set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
PBNG_TRACE=1 timeout 400 python scripts/quick_run.py 5 --reps 1 2>&1 | grep -v "^cd \|^fd " > gpurun_out/r20_q5.log
PBNG_TRACE=1 timeout 200 python scripts/quick_run.py 4 --reps 1 2>&1 | grep -v "^cd \|^fd " > gpurun_out/r20_q4.log
timeout 600 python bench.py --ablation > gpurun_out/r20_ablation.json 2> gpurun_out/r20_ablation.err; echo "abl rc=$?"
