"""The C++ host path (include/tkb/attention.hpp over the C ABI) through tools/tkb_mgpu, the
multi-GPU driver (one host thread per GPU, tkb_shard_range shards, no collective), run on
the GPUs this box has; --check verifies head 0 of every shard against the CPU oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "tkb_mgpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(EXE), reason="tools/tkb_mgpu not built")
@pytest.mark.parametrize("causal,dim", [(1, 128), (0, 64)])
def test_cpp_multi_gpu_driver(cuda_dev, causal, dim):
    import json

    r = subprocess.run([EXE, "--batch", "2", "--heads", "4", "--seq", "1024", "--dim", str(dim), "--causal",
                        str(causal), "--iters", "2", "--check"], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["gpus"] >= 1 and out["tflops_total"] > 0
    assert out["max_abs_err_head0"] <= 2e-2, out  # the north-star bar on O
