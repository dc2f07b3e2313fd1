"""The LCSF deadlock contract (reference: DeadlockError, lcsf.hpp:486-489; tested in
tests/test_lcsf.cpp:204-233): a consumer waiting on a ring slot that no producer fills must
not hang the GPU. mbar_wait's bounded spin traps (the self-test library is built with a
0.2 s bound instead of the product's 20 s), so the launch fails with a CUDA error. Runs in
a subprocess: a trap poisons the CUDA context of the process that hit it."""
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SCRIPT = textwrap.dedent("""
    import ctypes, sys, time
    sys.path.insert(0, {root!r})
    import torch
    from paper_2410_20399_b200 import _lib
    L = _lib.load_selftest()
    L.tkb_selftest_deadlock.argtypes = [ctypes.c_int, ctypes.c_void_p]
    done = torch.zeros(1, dtype=torch.int32, device="cuda")
    t0 = time.time()
    rc = L.tkb_selftest_deadlock({mode}, done.data_ptr())
    dt = time.time() - t0
    flag = int(done.item()) if rc == 0 else -1
    print(rc, flag, round(dt, 3))
""")


def _run(mode):
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, mode=mode)], capture_output=True, text=True,
                       timeout=120)
    return r


def test_ring_handoff_completes(cuda_dev):
    r = _run(1)
    assert r.returncode == 0, r.stderr
    rc, flag, _ = r.stdout.split()
    assert rc == "0" and flag == "1"


def test_missing_producer_traps_instead_of_hanging(cuda_dev):
    r = _run(0)
    # the trap surfaces as a launch failure (cudaErrorLaunchFailure / illegal instruction);
    # the process either reports the non-zero code or dies on the poisoned context
    if r.returncode == 0:
        rc, _, dt = r.stdout.split()
        assert rc != "0", r.stdout
        assert float(dt) < 30.0
