for v in s6a1 s6a2 s5a4 s6a1 s6a2 s5a4; do echo $v; TKB_LIB_PATH=build/libtkb_$v.so timeout 300 python tools/gemm_bench.py; done
TKB_LIB_PATH=build/libtkb_s6a2.so timeout 300 python -m pytest tests/test_gemm.py -x -q 2>&1 | tail -2
