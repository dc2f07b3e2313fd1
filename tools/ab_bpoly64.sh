for v in base bpoly2 bpoly3 base bpoly2; do TKB_LIB_PATH=build/libtkb_$v.so timeout 300 python tools/ab_bwd.py "16,16,4096,64,0;16,16,4096,64,1;64,16,1024,64,1"; done
