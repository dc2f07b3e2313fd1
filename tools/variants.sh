# usage: bash tools/variants.sh "<quick_bench args>" build/libA.so build/libB.so ...
args="$1"; shift
for lib in "$@"; do
  echo "== $lib"
  TKB_LIB_PATH=$PWD/$lib timeout 300 python tools/quick_bench.py $args 2>&1 | grep -v "^$"
done
