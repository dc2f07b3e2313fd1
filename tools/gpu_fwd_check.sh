# forward parity + quick timing of the current build
timeout 400 python -m pytest tests/test_attn_fwd_gpu.py -x -q 2>&1 | tail -15
timeout 200 python tools/quick_bench.py --shapes "16,16,4096,128;16,16,4096,64;4,16,16384,128;16,16,1024,128" 2>&1
