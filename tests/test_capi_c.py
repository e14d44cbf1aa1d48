"""The compiled C consumer (tests/c/capi_ref.c): a plain C99 program built
against the REFERENCE's own header (proj/include/mpsvd.h) and linked to
libmpsvd_b200.so (capi_ref), and the same source against include/mpsvd.h
(capi_own). Built by __graft_entry__.build() (paper_2603_11953_b200/build.py
build_c_consumers); the binaries travel to the GPU box with the repo.
Restates proj/tests/test_capi.cpp:24-126 for the thin-SVD surface."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "c", "_bin")
REF_HEADER = "/root/reference/proj/include/mpsvd.h"


def _binaries():
    names = ["capi_own"]
    # capi_ref is built wherever the reference header exists (the build
    # container); on the GPU box it arrives prebuilt with the snapshot
    if os.path.isfile(REF_HEADER) or os.path.exists(os.path.join(BIN, "capi_ref")):
        names.insert(0, "capi_ref")
    return names


def _run(name, *args, timeout=300):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout, cwd=BIN)


@pytest.mark.parametrize("name", _binaries())
def test_c_consumer_host_side(name):
    # no GPU needed: matrices, text IO, format_shortest, metrics on host
    # data; the compute entry points must fail with MPSVD_ERR_INTERNAL here
    M = pytest.importorskip("paper_2603_11953_b200")
    if M.device_available():
        pytest.skip("host-only mode checks the no-device error path")
    r = _run(name, "--host-only")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", _binaries())
def test_c_consumer_on_gpu(name):
    M = pytest.importorskip("paper_2603_11953_b200")
    if not M.device_available():
        pytest.skip("no CUDA device")
    r = _run(name)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
