"""The C++ drop-in (paper_2210_07297_b200/host/parplan_plan_gpu.cpp) against
the reference parplan::plan in one process (tests/cpp/test_drop_in.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_drop_in")


def test_cpp_drop_in_plan_equals_reference_plan():
    if not os.path.exists(BIN):
        pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ALL OK" in r.stdout


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("n_gpus", [2, 4])
def test_cpp_drop_in_multi_gpu_equals_reference_plan(n_gpus):
    """The same drop-in with one context driving n GPUs (LPT shards, NCCL
    all-gather of the top-k, per-record outputs gathered to the host):
    identical to the reference, hence to n_gpus = 1."""
    if not os.path.exists(BIN):
        pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    if _gpus() < n_gpus:
        pytest.skip(f"needs {n_gpus} GPUs")
    r = subprocess.run([BIN, str(n_gpus)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ALL OK" in r.stdout and f"n_gpus = {n_gpus}" in r.stdout
