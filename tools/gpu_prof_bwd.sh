# ncu full of the backward kernels (one step after a warm step) + the cycle trace
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dkdvp|attn_bwd_dq" -s 2 -c 2 \
    -o gpurun_out/bwd_full -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_bwd.log 2>&1; echo ncu rc=$?
timeout 300 python tools/trace_bwd.py 16,16,4096,128,1 > gpurun_out/trace_bwd.log 2>&1; echo trace rc=$?
tail -40 gpurun_out/trace_bwd.log
