# BASELINE configs[0] through bench.py with the forward's task shape forced to two tiles (2) or
# chosen by problem size (0: one-tile tasks here), alternating
for t in 2 0 2 0; do
python - "$t" <<'PY'
import contextlib, io, json, sys
t = int(sys.argv[1])
sys.argv = ["bench.py", "--batch", "1", "--heads", "8", "--seq", "1024", "--head-dim", "64", "--causal", "0",
            "--pass", "fwd", "--no-e2e"]
sys.path.insert(0, ".")
from paper_2410_20399_b200 import attention as A
import bench
A.debug_set_fwd_task_tiles(t)
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
d = json.loads([l for l in buf.getvalue().splitlines() if l.startswith("{")][-1])
print("tiles", t, "value", round(d["value"], 1), "us/step", round(d["ms_per_step"] * 1e3, 1), "isolated us",
      round(d["roofline"]["per_kernel"]["attn_fwd"]["us"], 1), flush=True)
PY
done
