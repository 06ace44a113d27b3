set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_atoms scripts/ubench_atoms.cu && /tmp/ubench_atoms > gpurun_out/r8_ubench.json
cat gpurun_out/r8_ubench.json
export PBNG_TRACE=1
timeout 400 python scripts/quick_run.py 5 --reps 1 > gpurun_out/r8_q5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg_win -s 45 -c 1 -o gpurun_out/r8_prof_win5 python scripts/quick_run.py 5 --reps 1 > gpurun_out/r8_ncu.log 2>&1
echo "ncu rc=$?"
