# round-2 measurement pass: launch list + ncu full of the bench step, N=768 ncu (dram vs
# algorithmic), C1 line, GEMM vs cuBLAS, configs[3] sweep, fused-rotary A/B.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"attn_fwd_template|attn_bwd_dkdv_template|attn_bwd_dq_template|bwd_prep" -s 4 -c 4 \
    -o gpurun_out/r2_full -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --kernel-name-base demangled -k regex:"attn_fwd_template|attn_bwd|bwd_prep" -s 4 -c 4 --csv \
    --log-file gpurun_out/r2_n768.csv python tools/profile_step.py --shape 16,16,768,128 --steps 2 > gpurun_out/ncu_768.log 2>&1
echo n768 rc=$?
timeout 300 python bench.py --batch 1 --heads 8 --seq 1024 --head-dim 64 --causal 0 --pass fwd --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/r2_c1.log 2>&1
echo c1 rc=$?; tail -1 gpurun_out/r2_c1.log
timeout 600 python tools/gemm_bench.py > gpurun_out/r2_gemm.log 2>&1; echo gemm rc=$?; tail -12 gpurun_out/r2_gemm.log
timeout 900 python tools/sweep.py > gpurun_out/r2_sweep.log 2>&1; echo sweep rc=$?; tail -5 gpurun_out/r2_sweep.log
