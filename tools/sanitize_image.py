"""Small runs of the image-stream paths for compute-sanitizer: init_image,
frame_normalize_auto (current state and a captured slot, fp32 and fp64),
Pipeline.run_images on two handles, and a pre-faulted pageable download."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2102_10340_b200 as fhn  # noqa: E402

rng = np.random.default_rng(0)
for prec in ("single", "double"):
    with fhn.Simulator(64, 96, precision=prec) as s:
        s.init_image(rng.integers(0, 256, (64, 96), dtype=np.uint8), 1.0)
        s.advance(9)
        s.frame_normalize_auto()
        s.frames_reserve(1)
        s.frame_capture(0)
        s.frame_normalize_auto(slot=0)
imgs = [rng.integers(0, 256, 96 * 128, dtype=np.uint8) for _ in range(3)]
outs = [np.empty(96 * 128, np.uint8) for _ in imgs]
pipe = fhn.Pipeline(96, 128, depth=2)
pipe.run_images([(a.ctypes.data, b.ctypes.data) for a, b in zip(imgs, outs)], 7, 1.0)
pipe.close()
with fhn.Simulator(2048, 2048, levels=4) as s:  # 16 MiB planes x 2: the pre-fault threshold is 32 MiB per plane
    s.init(1, 42)
with fhn.Simulator(128, 128, batch=1024, levels=4) as s:  # 64 MiB planes: pre-faulted download
    s.init(1, 42)
    s.advance(4)
    s.download()
    s.frames_reserve(1)
    s.frame_capture(0)
    s.frame_download(0)
print("sanitize image paths done")
