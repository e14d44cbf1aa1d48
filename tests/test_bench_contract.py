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

    def __init__(self, gram_kernel=0, av_kernel=1):
        self.gram_kernel, self.av_kernel = gram_kernel, av_kernel


def test_phase_rooflines_f32_units_and_fractions():
    # K1 (DMMA): m n (n+1) flops against the fp64 tensor peak; K7 on HBM
    cfg = inputs.CONFIGS["c2"]
    med = {"gram": 0.2, "eigen": 0.25, "compute_u": 0.13}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info(0, 1))
    g = ph["gram"]
    assert g["bound"] == "tensor" and g["unit"] == "TFLOP/s" and g["ncu_kernel"] == "gram_f32_diag"
    assert g["achieved"] == pytest.approx(cfg.m * cfg.n * (cfg.n + 1) / 0.2e-3 / 1e12)
    assert g["frac"] == pytest.approx(g["achieved"] / 37.0)
    u = ph["compute_u"]
    assert u["bound"] == "hbm" and u["achieved"] == pytest.approx(2 * cfg.m * cfg.n * 4 / 0.13e-3 / 1e9)
    assert u["ncu_kernel"] == "av_tc_tmem_f32"
    assert ph["eigen"]["bound"] == "latency"


def test_phase_rooflines_k1z_against_int8_peak():
    # K1z: 12 int8 MMAs (M = N = 128, K = 32) per 32-row chunk against the
    # kind::i8 peak, plus its A stream against HBM
    cfg = inputs.CONFIGS["c4"]
    med = {"gram": 24.0, "eigen": 2.7, "compute_u": 14.5}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info(1, 1))
    g = ph["gram"]
    assert g["ncu_kernel"] == "gram_f32_ozaki" and g["unit"] == "TOPS"
    assert g["achieved"] == pytest.approx(cfg.m * 12 * 2 * 128 * 128 / 24e-3 / 1e12)
    assert g["peak"] == pytest.approx(bench.I8_TOPS)
    assert g["hbm_achieved_gbs"] == pytest.approx(cfg.m * cfg.n * 4 / 24e-3 / 1e9)


def test_phase_rooflines_dd_uses_c_dd_10():
    # K2 (Dot2): c_dd = 10 fp64 operations per multiply-add
    cfg = inputs.CONFIGS["c5"]
    med = {"gram": 1400.0, "eigen": 800.0, "compute_u": 270.0}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info(2, 2))
    g = ph["gram"]
    assert g["achieved"] == pytest.approx(cfg.m * cfg.n * (cfg.n + 1) / 2 * 10 / 1.4 / 1e12)
    assert g["peak"] == pytest.approx(bench.DFMA_TFLOPS / 2)
    assert ph["compute_u"]["bound"] == "tensor"


def test_phase_rooflines_dd_ozaki_against_int8_peak():
    # K2z: 66 int8 digit products per multiply-add against the measured
    # kind::i8 tensor peak; U on DMMA (c5's dominant phase: the line's
    # headline roofline must exist for it)
    cfg = inputs.CONFIGS["c5"]
    med = {"gram": 236.0, "eigen": 800.0, "compute_u": 270.0}
    ph = bench.phase_rooflines(cfg, cfg.m, cfg.n, med, 37.0, 6555.2, _Info(3, 2))
    g = ph["gram"]
    assert g["achieved"] == pytest.approx(2 * 66 * cfg.m * cfg.n * (cfg.n + 1) / 2 / 0.236 / 1e12)
    assert g["peak"] == pytest.approx(bench.I8_TOPS)
    assert 4700 < bench.I8_TOPS < 4800
    assert ph["compute_u"]["ncu_kernel"] == "av_dmma_f64"


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
