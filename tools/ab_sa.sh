python -m pytest tests/test_attn_bwd_gpu.py tests/test_gqa_gpu.py -x -q 2>&1 | tail -2
for v in sa2 sa3 sa4 sa2 sa4; do TKB_LIB_PATH=build/libtkb_$v.so timeout 300 python tools/ab_bwd.py "16,16,4096,64,0;16,16,4096,64,1;64,16,1024,64,1"; done
python tools/trace_bwd_boundary.py 16,16,4096,64,0 2>&1 | head -3
