"""bench.py's JSON contract pieces that need no GPU: the per-phase roofline
arithmetic, the shared config of both arms, and the reference arm's line."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import workloads as inputs  # noqa: E402


class _Info:
    rotations = 1000


def test_phase_rooflines_f32_units_and_fractions():
    cfg = inputs.CONFIGS["c2"]
    med = {"gram": 0.2, "eigen": 0.25, "compute_u": 0.13}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info())
    g = ph["gram"]
    assert g["bound"] == "tensor" and g["unit"] == "TFLOP/s"
    assert g["achieved"] == pytest.approx(cfg.m * cfg.n * (cfg.n + 1) / 0.2e-3 / 1e12)
    assert g["frac"] == pytest.approx(g["achieved"] / 37.0)
    u = ph["compute_u"]
    assert u["bound"] == "hbm" and u["achieved"] == pytest.approx(2 * cfg.m * cfg.n * 4 / 0.13e-3 / 1e9)
    assert ph["eigen"]["bound"] == "latency"


def test_phase_rooflines_dd_uses_c_dd_10(monkeypatch):
    # K2 (Dot2, forced): c_dd = 10 fp64 operations per multiply-add
    monkeypatch.setenv("MPSVD_DD_GRAM", "dot2")
    cfg = inputs.CONFIGS["c5"]
    med = {"gram": 1400.0, "eigen": 800.0, "compute_u": 270.0}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info())
    g = ph["gram"]
    assert g["achieved"] == pytest.approx(cfg.m * cfg.n * (cfg.n + 1) / 2 * 10 / 1.4 / 1e12)
    assert g["peak"] == pytest.approx(bench.DFMA_TFLOPS / 2)
    assert ph["compute_u"]["bound"] == "tensor"


def test_phase_rooflines_dd_ozaki_against_int8_peak(monkeypatch):
    # K2z (the engine's choice from 4096 rows): 66 int8 digit products per
    # multiply-add against the measured kind::i8 tensor peak
    monkeypatch.delenv("MPSVD_DD_GRAM", raising=False)
    cfg = inputs.CONFIGS["c5"]
    med = {"gram": 236.0, "eigen": 800.0, "compute_u": 270.0}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info())
    g = ph["gram"]
    assert g["achieved"] == pytest.approx(2 * 66 * cfg.m * cfg.n * (cfg.n + 1) / 2 / 0.236 / 1e12)
    assert g["peak"] == pytest.approx(bench.I8_TOPS)
    assert 4700 < bench.I8_TOPS < 4800
    assert not bench.ozaki_gram(4095) and bench.ozaki_gram(4096)


@pytest.mark.parametrize("name,world", [("c2", 1), ("c2", 8), ("c4", 4), ("c5", 2)])
def test_config_dict_weak_and_strong(name, world):
    cfg = inputs.CONFIGS[name]
    d = bench.config_dict(cfg, world)
    assert d["workload"] == name and d["n"] == cfg.n and d["parallelism"] == f"rows{world}"
    assert d["m"] == (cfg.m * world if name == "c2" else cfg.m)  # c2 weak, the rest strong


def test_reference_arm_line_shape():
    env = dict(os.environ, RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["workload"] == "c1" and line["cpu_baseline"]["cores"] >= 1


def test_reference_arm_other_ranks_print_nothing():
    env = dict(os.environ, RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0 and out.stdout.strip() == ""
