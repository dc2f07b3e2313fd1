for sh in 64,16,16,1024,128,1,0 16,16,16,4096,128,1,0 16,16,16,4096,128,0,0; do
  for v in warm0 fd warm0 fd; do SECS=2 TKB_LIB_PATH=build/libtkb_$v.so python tools/ab_fwd.py $sh; done
done
TKB_LIB_PATH=build/libtkb_ftracefd.so python tools/trace_fwd.py 16,16,4096,128,1 > gpurun_out/trace_fwd4k_fd.log 2>&1
