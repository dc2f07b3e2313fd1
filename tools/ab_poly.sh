for v in default poly0 poly2; do
  if [ $v = default ]; then unset TKB_LIB_PATH; else export TKB_LIB_PATH=build/libtkb_$v.so; fi
  echo "== $v"; python tools/quick_bench.py --bwd --only-causal --shapes "16,16,4096,128;16,16,4096,64" --soak 3 2>&1 | grep bwd
done
