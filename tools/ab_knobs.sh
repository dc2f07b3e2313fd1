for sh in 16,16,16,4096,128,1,0 16,16,16,4096,128,0,0 64,16,16,1024,128,1,0; do
  for v in base pc1 pc4 poly1 poly3 base; do SECS=2 TKB_LIB_PATH=build/libtkb_$v.so python tools/ab_fwd.py $sh; done
done
for v in base bpoly0 bpoly2 base; do TKB_LIB_PATH=build/libtkb_$v.so timeout 300 python tools/ab_bwd.py "16,16,4096,128,1;16,16,4096,128,0"; done
