python -m pytest tests/test_attn_bwd_gpu.py tests/test_gqa_gpu.py tests/test_varlen_gpu.py tests/test_fuzz_gpu.py -x -q 2>&1 | tail -2
for v in base preq base preq; do TKB_LIB_PATH=build/libtkb_$v.so timeout 300 python tools/ab_bwd.py "16,16,4096,128,1;16,16,4096,128,0;64,16,1024,128,1;16,16,4096,64,1"; done
TKB_LIB_PATH=build/libtkb_preq.so python tools/trace_dq.py 16,16,4096,128,1 2>&1 | head -4
