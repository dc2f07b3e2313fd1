set -x
for sh in 64,16,16,1024,128,1,0 16,16,16,4096,128,1,0 16,16,16,4096,128,0,0; do
  for v in orig warm0 warm1 warm2 warm3 orig warm2; do SECS=2 TKB_LIB_PATH=build/libtkb_$v.so python tools/ab_fwd.py $sh; done
done
TKB_LIB_PATH=build/libtkb_ftrace.so python tools/trace_fwd.py 16,16,4096,128,1 > gpurun_out/trace_fwd4k_w2.log 2>&1
TKB_LIB_PATH=build/libtkb_ftrace0.so python tools/trace_fwd.py 16,16,4096,128,1 > gpurun_out/trace_fwd4k_w0.log 2>&1
