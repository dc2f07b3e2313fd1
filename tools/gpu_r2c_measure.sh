# round-2c measurement pass: launch list + ncu full of the bench step, smoke, bench line, C1 line,
# configs[3] sweep (outputs gpurun_out/r2c_*; summarised into profiles/ by tools/ncu_summary.py)
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv \
    --log-file gpurun_out/r2c_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"attn_fwd_template|attn_bwd_dkdv_template|attn_bwd_dq_template|bwd_prep" -s 4 -c 4 \
    -o gpurun_out/r2c_full -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench rc=$?
timeout 300 python bench.py --batch 1 --heads 8 --seq 1024 --head-dim 64 --causal 0 --pass fwd --steps 50 --warmup 10 \
    --no-cpu-baseline > gpurun_out/r2c_c1.log 2>&1; echo c1 rc=$?
timeout 1200 python tools/sweep.py > gpurun_out/r2c_sweep.log 2>&1; echo sweep rc=$?
