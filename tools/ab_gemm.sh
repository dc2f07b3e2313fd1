timeout 300 python -m pytest tests/test_gemm.py -x -q 2>&1 | tail -3
for v in gsingle gpair gsingle gpair; do echo $v; TKB_LIB_PATH=build/libtkb_$v.so timeout 300 python tools/gemm_bench.py; done
