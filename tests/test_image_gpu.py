"""The edge-detection image stream on the device: normalize_frame with the
plane's own min/max (rdcnn_sim_frame_normalize_auto) and Pipeline.run_images,
checked against the host normalize_frame (imageio, itself checked against the
reference's, tests/test_cli_io.py) on the downloaded state."""
import numpy as np
import pytest

import paper_2102_10340_b200 as fhn
from paper_2102_10340_b200 import imageio

pytestmark = pytest.mark.gpu


def _pixels(rows, cols, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, (rows, cols), dtype=np.uint8)


@pytest.mark.parametrize("precision", ("single", "double"))
@pytest.mark.parametrize("rows,cols", [(64, 128), (37, 96), (512, 512)])
def test_normalize_auto_equals_host(precision, rows, cols):
    with fhn.Simulator(rows, cols, precision=precision) as sim:
        sim.init_image(_pixels(rows, cols, 1), 1.0)
        sim.advance(17)
        img, lo, hi = sim.frame_normalize_auto()
        u, _ = sim.download()
        want, wlo, whi = imageio.normalize_frame(u.reshape(rows, cols))
        assert (lo, hi) == (wlo, whi)
        assert np.array_equal(img, want)
        # a captured slot, and the fixed-range call with the same bounds
        sim.frames_reserve(1)
        sim.frame_capture(0)
        img2, lo2, hi2 = sim.frame_normalize_auto(slot=0)
        assert (lo2, hi2) == (lo, hi) and np.array_equal(img2, img)
        assert np.array_equal(sim.frame_normalize(-1, 0, lo, hi), img)


def test_normalize_auto_flat_plane():
    with fhn.Simulator(32, 64) as sim:
        sim.init_image(np.full((32, 64), 77, np.uint8), 1.0)
        img, lo, hi = sim.frame_normalize_auto()
        assert lo == hi and (img == 128).all()


def test_normalize_auto_signed_values():
    rows, cols = 48, 64
    rng = np.random.default_rng(4)
    u = rng.normal(0.0, 3.0, rows * cols).astype(np.float32)
    u[5] = -0.0
    u[6] = np.float32(-7.5e-39)  # subnormal
    with fhn.Simulator(rows, cols) as sim:
        sim.upload(u, np.zeros_like(u))
        img, lo, hi = sim.frame_normalize_auto()
    want, wlo, whi = imageio.normalize_frame(u.reshape(rows, cols))
    assert (lo, hi) == (wlo, whi) and np.array_equal(img, want)


def test_run_images_equals_sequential():
    rows, cols, steps = 96, 128, 30
    imgs = [_pixels(rows, cols, s) for s in range(5)]
    outs = [np.empty(rows * cols, np.uint8) for _ in imgs]
    pipe = fhn.Pipeline(rows, cols, depth=2)
    pipe.set_params(fhn.Gene())
    bad = pipe.run_images([(im.ctypes.data, o.ctypes.data) for im, o in zip(imgs, outs)], steps, 1.0)
    pipe.close()
    assert not bad.any()
    for im, o in zip(imgs, outs):
        with fhn.Simulator(rows, cols) as sim:
            sim.init_image(im, 1.0)
            sim.advance(steps)
            u, _ = sim.download()
        want, _, _ = imageio.normalize_frame(u.reshape(rows, cols))
        assert np.array_equal(o.reshape(rows, cols), want)
