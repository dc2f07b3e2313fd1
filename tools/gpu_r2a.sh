# round-2 GPU pass: full GPU tests, smoke, default bench, configs[4] full size on one GPU
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log
timeout 900 python bench.py --batch 32 --heads 32 --seq 16384 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5 rc=$?; tail -1 gpurun_out/bench_c5.log
