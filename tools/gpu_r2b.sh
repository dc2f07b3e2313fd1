set -x
timeout 300 python -m pytest tests/test_primitives_gpu.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu -x -k "bwd or fuzz or gqa or long or pairs or cpp or smoke" 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2b.log 2>&1; tail -1 gpurun_out/bench_r2b.log
