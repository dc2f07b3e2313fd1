# usage: bash tools/clk_probe.sh <lib.so> [quick_bench args...]
# Runs tools/quick_bench.py while sampling nvidia-smi every 100 ms; prints the bench lines and
# the median SM clock / power over the samples drawing > 300 W (the loaded ones).
lib=$1; shift
f=$(mktemp)
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > $f &
P=$!
TKB_LIB_PATH=$PWD/$lib timeout 300 python tools/quick_bench.py "$@" 2>&1 | grep "^bwd\|^fwd\|Error"
kill $P
python3 - "$f" <<'PY'
import sys, statistics
rows = [tuple(float(x) for x in l.split(",")) for l in open(sys.argv[1]) if l.strip()]
hot = [r for r in rows if r[1] > 300]
if hot:
    print("loaded samples %d: median sm %.0f MHz, median power %.0f W" % (
        len(hot), statistics.median(r[0] for r in hot), statistics.median(r[1] for r in hot)))
PY
