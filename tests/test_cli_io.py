"""Front end and image I/O (§8f4): manifest text, PGM/PNG bytes and frame
normalisation against the reference's own code (oracle/_ref), and the CLI's
reference-shaped behaviour (rdcnn_cli.cpp; acceptance 10 and 11) on a GPU."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import REF_SO
from paper_2102_10340_b200 import imageio
from paper_2102_10340_b200.cli import manifest_text, parse_manifest
from paper_2102_10340_b200.engine import Gene, RunConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(REF_SO)


@pytest.fixture(scope="module")
def ref():
    if not HAVE_REF:
        pytest.skip("oracle/_ref not built")
    return ctypes.CDLL(REF_SO)


def test_manifest_matches_reference(ref):
    f = ref.ref_manifest_text
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long, ctypes.c_int,
                  ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]
    for g, cfg in [(Gene(), RunConfig(nn=64, nm=64, iter_max=200, nssp=5, seed=42)),
                   (Gene(a=-0.05, Du=0.0001, dt=1e-5, ka=2.5), RunConfig(init_mode=2, nn=30, nm=17, iter_max=77,
                                                                        nssp=7, seed=123456789,
                                                                        precision="double"))]:
        g8 = np.asarray(g.to_vector() + [g.ka], np.float64)
        buf = ctypes.create_string_buffer(4096)
        assert f(g8.ctypes.data, cfg.init_mode, cfg.nn, cfg.nm, cfg.iter_max, cfg.nssp, cfg.seed, b"parallel",
                 int(cfg.precision == "double"), buf, 4096) == 0
        assert manifest_text(g, cfg, backend="parallel") == buf.value.decode()
        g2, cfg2 = parse_manifest(manifest_text(g, cfg))
        assert g2 == g and (cfg2.nn, cfg2.nm, cfg2.iter_max, cfg2.nssp, cfg2.seed, cfg2.precision) == \
            (cfg.nn, cfg.nm, cfg.iter_max, cfg.nssp, cfg.seed, cfg.precision)


def test_png_and_pgm_bytes_match_reference(ref, tmp_path):
    f = ref.ref_write_image
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    rng = np.random.default_rng(4)
    for shape in [(3, 5), (64, 48), (17, 130)]:
        img = rng.integers(0, 256, shape, dtype=np.uint8)
        img[: shape[0] // 2] = np.arange(shape[1], dtype=np.uint8)[None, :]  # compressible part
        for png in (0, 1):
            rp = str(tmp_path / f"r{png}")
            assert f(rp.encode(), shape[0], shape[1], img.ctypes.data, png) == 0
            mp = str(tmp_path / f"m{png}")
            (imageio.write_png if png else imageio.write_pgm)(mp, img)
            assert open(rp, "rb").read() == open(mp, "rb").read()
            back = imageio.read_png(mp) if png else imageio.read_pgm(mp)
            assert np.array_equal(back, img)


def test_png_reader_handles_all_filters(tmp_path):
    import struct
    import zlib
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (6, 9), dtype=np.uint8)
    rows = []
    prev = np.zeros(9, np.int64)
    for i, ftype in enumerate([0, 1, 2, 3, 4, 1]):
        x = img[i].astype(np.int64)
        a = np.concatenate([[0], x[:-1]])
        c = np.concatenate([[0], prev[:-1]])
        if ftype == 0:
            f = x
        elif ftype == 1:
            f = x - a
        elif ftype == 2:
            f = x - prev
        elif ftype == 3:
            f = x - (a + prev) // 2
        else:
            f = x - np.array([imageio._paeth(int(a[k]), int(prev[k]), int(c[k])) for k in range(9)])
        rows.append(bytes([ftype]) + bytes((f & 0xFF).astype(np.uint8)))
        prev = x
    raw = b"".join(rows)
    data = (b"\x89PNG\r\n\x1a\n" + imageio._chunk(b"IHDR", struct.pack(">IIBBBBB", 9, 6, 8, 0, 0, 0, 0))
            + imageio._chunk(b"IDAT", zlib.compress(raw)) + imageio._chunk(b"IEND", b""))
    p = tmp_path / "f.png"
    p.write_bytes(data)
    assert np.array_equal(imageio.read_png(str(p)), img)


def test_normalize_frame_matches_reference(ref):
    f = ref.ref_normalize_frame_f32
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                  ctypes.POINTER(ctypes.c_double)]
    rng = np.random.default_rng(9)
    for x in [rng.standard_normal((40, 50)).astype(np.float32),
              np.linspace(-1, 1, 255 * 4 + 1, dtype=np.float32).reshape(1, -1)[:, :1020].reshape(20, 51),
              np.full((5, 5), 0.25, np.float32)]:
        out = np.empty(x.size, np.uint8)
        lo, hi = ctypes.c_double(), ctypes.c_double()
        f(x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data, ctypes.byref(lo), ctypes.byref(hi))
        mine, mlo, mhi = imageio.normalize_frame(x)
        assert np.array_equal(mine.reshape(-1), out) and (mlo, mhi) == (lo.value, hi.value)


def test_lround_is_half_away_from_zero():
    y = np.array([0.5, 1.5, 2.5, -0.5, 0.49999999999999994, 254.5, 2.0 ** 52 + 1])
    assert imageio.lround(y).tolist() == [1, 2, 3, -1, 0, 255, 2 ** 52 + 1]


def test_cli_rejects_bad_flags_and_cpu_backends():
    from paper_2102_10340_b200.cli import main
    assert main(["simulate", "--size", "2", "--iters", "10", "--nssp", "3"]) == 1
    assert main(["simulate", "--backend", "parallel", "--size", "16", "--iters", "10", "--nssp", "1"]) == 1
    assert main(["sweep", "--x", "du:0.1"]) == 1


# --- GPU: the front end end to end ---------------------------------------------

def _cli(args, cwd):
    return subprocess.run([sys.executable, "-m", "paper_2102_10340_b200", *args], cwd=cwd, capture_output=True,
                          text=True, env={**os.environ, "PYTHONPATH": ROOT})


@pytest.mark.gpu
def test_cli_simulate_kat_and_replay(tmp_path):
    """acceptance 10: manifest replay gives equal digests and identical frames."""
    a = _cli(["simulate", "--typ", "1", "--size", "64", "--iters", "200", "--nssp", "5", "--seed", "42",
              "--out", str(tmp_path / "a")], ROOT)
    assert a.returncode == 0, a.stderr
    assert "checksum= ced829150965fba9" in a.stdout
    assert "FHN Calculation: 64 x 64 mesh" in a.stdout and "199, (elapsed:" in a.stdout
    b = _cli(["simulate", "--manifest", str(tmp_path / "a" / "manifest.txt"), "--out", str(tmp_path / "b")], ROOT)
    assert b.returncode == 0, b.stderr
    assert "checksum= ced829150965fba9" in b.stdout
    for name in ("final_u.png", "final_v.pgm", "frame_000200_u.pgm"):
        assert (tmp_path / "a" / name).read_bytes() == (tmp_path / "b" / name).read_bytes()


@pytest.mark.gpu
def test_cli_blowup_exit_code(tmp_path):
    """acceptance 11: dt=100 -> exit 2, stderr names the iteration, no result files."""
    r = _cli(["simulate", "--typ", "1", "--size", "32", "--iters", "1000", "--nssp", "1", "--seed", "42",
              "--dt", "100", "--out", str(tmp_path / "blow")], ROOT)
    assert r.returncode == 2 and "iteration" in r.stderr
    assert (tmp_path / "blow" / "manifest.txt").exists()
    assert not (tmp_path / "blow" / "final_u.png").exists()


@pytest.mark.gpu
def test_cli_sweep_and_bench(tmp_path):
    r = _cli(["sweep", "--x", "du:0.02,0.3", "--y", "dv:0.5,1.0,5.0", "--size", "32", "--iters", "200", "--nssp",
              "5", "--seed", "42", "--out", str(tmp_path / "sw")], ROOT)
    assert r.returncode == 0, r.stderr
    import json
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["sweeps"][0]["labels_csv"]
    assert (tmp_path / "sw" / "labels.csv").read_text() == gold
    r = _cli(["bench", "--sizes", "64,128", "--iters", "200", "--reps", "2", "--out", str(tmp_path / "bn")], ROOT)
    assert r.returncode == 0, r.stderr
    csv = (tmp_path / "bn" / "bench.csv").read_text().splitlines()
    assert csv[0] == "backend,hardware,n,iters,seconds,mcells_per_s,ns_per_cell_iter,checksum"
    assert csv[1].startswith("cuda,b200,64,200,") and csv[1].endswith(",ced829150965fba9")
