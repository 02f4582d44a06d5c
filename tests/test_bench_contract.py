"""bench.py keeps the driver's JSON contract (one line; metric/value/unit/
n_gpus/steps/warmup/ms_per_step/higher_is_better/scaling/vs_baseline/dtype/
data/config, plus roofline, cpu_baseline, e2e, gpu_launches, clocks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    """The reference arm (the reference's own parallel backend on the host)."""
    d = run_bench("--impl", "reference", "--size", "64", "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Mcell-updates/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_uses_every_host_core():
    """torchrun exports OMP_NUM_THREADS=1 to each rank; the reference arm must
    still run the reference's parallel backend on every usable host core."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    d = run_bench("--impl", "reference", "--size", "64", "--steps", "1", "--warmup", "1", env=env)
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_reference_arm_prints_our_arms_config():
    """Both arms describe the same workload (config) so the driver compares
    like with like; the reference's bounded sample is recorded beside it."""
    d = run_bench("--impl", "reference", "--size", "64", "--steps", "2", "--warmup", "1")
    c = d["config"]
    assert c["iterations_per_step"] == 10000 and c["rows"] == 64 and c["parallelism"] == "single"
    assert c["workload"].startswith("cfg2") and c["levels_per_launch"] == 4 and c["mode"] == "strict"
    cb = d["cpu_baseline"]
    assert cb["iterations_per_step_sampled"] >= 1 and ".." in cb["iterations_timed"]
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    args = argparse.Namespace(workload="cfg2", size=64, iters_per_step=None, levels=4, mode="strict",
                              slab=False, ring=False, devices=None, transport="auto")
    wl = bench.Workload(args, 1)
    assert bench.config_dict(wl, args, 1, *bench.predicted_layout(wl, args, 1)) == c


def test_reference_arm_ring_mode_config():
    """--devices without torchrun: the reference arm runs the same global
    lattice (weak scaling: one 64-row slab per entry) and says so."""
    d = run_bench("--impl", "reference", "--size", "64", "--steps", "1", "--warmup", "1", "--devices", "0,0")
    assert d["config"]["rows"] == 128 and d["config"]["parallelism"] == "slab2"
    assert d["config"]["transport"] == "p2p"


@pytest.mark.gpu
def test_our_arm_ring_mode():
    """Single-process multi-GPU mode (rdcnn_ring_*), here two slabs on the
    one device: the line records the slabs, devices and launches."""
    d = run_bench("--devices", "0,0", "--size", "256", "--steps", "2", "--warmup", "3", "--iters-per-step", "40",
                  "--no-cpu-baseline", "--e2e-steps", "1")
    assert d["n_gpus"] == 1 and d["slabs"] == 2 and d["devices"] == [0, 0]
    assert d["config"]["parallelism"] == "slab2" and d["config"]["rows"] == 512
    assert d["gpu_launches"] == 2 * 2 * 40 // 4 and d["value"] > 0
    assert d["e2e"]["device_ms_per_step"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 2 * 4 * 512 * 256


@pytest.mark.gpu
def test_our_arm_contract():
    d = run_bench("--size", "512", "--steps", "3", "--warmup", "3", "--iters-per-step", "40",
                  "--no-cpu-baseline", "--e2e-steps", "1")
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["higher_is_better"] is True
    # the binding roof leads: the K-blocked stencil is FP32-pipe bound
    r = d["roofline"]
    assert r["bound"] == "fp32" and r["unit"] == "TFLOP/s" and r["peak"] > 0 and 0 < r["frac"] < 1.2
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 4 * 512 * 512 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert d["config"]["workload"].startswith("cfg2")
    assert 0 < r["frac"] <= r["frac_at_median_clock"] + 1e-9
    assert r["hbm"]["compulsory_frac"] < 1.2 and r["hbm"]["effective_gbs"] > r["hbm"]["compulsory_gbs"]
    assert d["e2e"]["device_ms_per_step"] > 0 and "copy_and_host_ms_per_step" in d["e2e"]
    # BASELINE.md §1 publishes PyCUDA/P100 at N=512 (7581 Mcells/s): vs_baseline is value / that
    assert d["vs_baseline"] == pytest.approx(d["value"] / 7581.0, rel=1e-3) and "P100" in d["vs_baseline_basis"]


@pytest.mark.gpu
def test_our_arm_slab_contract():
    d = run_bench("--slab", "--size", "512", "--steps", "2", "--warmup", "3", "--iters-per-step", "40",
                  "--no-cpu-baseline", "--e2e-steps", "1")
    assert d["config"]["transport"] == "p2p" and d["value"] > 0


@pytest.mark.gpu
def test_our_arm_image_stream_e2e():
    """cfg3 (edge detection over a stream of images): the e2e runs three images
    in flight through engine.Pipeline; cfg2 (one evolving lattice) runs one."""
    d = run_bench("--workload", "cfg3", "--size", "512", "--steps", "2", "--warmup", "3",
                  "--iters-per-step", "20", "--no-cpu-baseline", "--e2e-steps", "4")
    assert d["e2e"]["lattices_in_flight"] == 3 and d["e2e"]["steps"] == 4 and d["e2e"]["value"] > 0
    # per image: its 8-bit pixels up, the normalised 8-bit edge map (+ its min/max) back
    assert d["e2e"]["h2d_bytes_per_step"] == 512 * 512
    assert d["e2e"]["d2h_bytes_per_step"] == 512 * 512 + 16
    assert "run_images" in d["e2e"]["path"]
    # the float-state stream on request: both planes each way
    d = run_bench("--workload", "cfg3", "--size", "512", "--steps", "2", "--warmup", "3",
                  "--iters-per-step", "20", "--no-cpu-baseline", "--e2e-steps", "4", "--e2e-states")
    assert d["e2e"]["lattices_in_flight"] == 3 and d["e2e"]["h2d_bytes_per_step"] == 2 * 4 * 512 * 512
    d = run_bench("--size", "512", "--steps", "2", "--warmup", "3", "--iters-per-step", "40",
                  "--no-cpu-baseline", "--e2e-steps", "2")
    assert d["e2e"]["lattices_in_flight"] == 1
