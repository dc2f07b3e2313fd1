python -m pytest tests/test_gqa_gpu.py tests/test_attn_bwd_gpu.py tests/test_varlen_gpu.py tests/test_fuzz_gpu.py -x -q 2>&1 | tail -3
for v in base split2 base split2; do echo $v; TKB_LIB_PATH=build/libtkb_$v.so python tools/gqa_bench.py; done
