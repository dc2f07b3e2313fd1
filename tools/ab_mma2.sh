python -m pytest tests/test_attn_fwd_gpu.py tests/test_rotary.py tests/test_gqa_gpu.py tests/test_varlen_gpu.py tests/test_fuzz_gpu.py -x -q 2>&1 | tail -3
for sh in 64,16,16,1024,128,1,0 16,16,16,4096,128,1,0 16,16,16,4096,128,0,0 16,16,16,4096,128,1,1; do
  for v in fd mma2 fd mma2; do SECS=2 TKB_LIB_PATH=build/libtkb_$v.so python tools/ab_fwd.py $sh; done
done
TKB_LIB_PATH=build/libtkb_ftrace2.so python tools/trace_fwd.py 16,16,4096,128,1 > gpurun_out/trace_fwd4k_mma2.log 2>&1
