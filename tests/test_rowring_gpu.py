"""The row-ring kernel (fhn_rowring.cuh: a thread-block cluster spans a whole
torus row, neighbours through shared memory and DSMEM st.async, no halo
lanes) against the wavefront kernel, bit for bit.  It is off by default
(measured slower, profiles/README.md), so each case runs in a subprocess with
RDCNN_ROWRING=1 and RDCNN_RR_M pinned, and the wavefront result comes from a
subprocess with RDCNN_ROWRING=0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import ctypes, json, sys
sys.path.insert(0, ROOT)
import paper_2102_10340_b200 as fhn
rows, cols, typ, steps, gene = ARGS
out = {}
with fhn.Simulator(rows, cols, 1, levels=4, mode="strict", persistent=-1) as sim:
    sim.set_params(fhn.Gene(**gene))
    sim.init(typ, 42)
    bad = (ctypes.c_long * 1)()
    out["rc"] = int(sim._lib.rdcnn_sim_advance(sim._h, steps, bad))
    out["bad"] = int(bad[0])
    out["checksum"] = "%016x" % int(sim.checksums()[0])
    out["launches"] = sim.launch_count()
print("RESULT " + json.dumps(out))
"""


def run(env_extra, args):
    env = dict(os.environ)
    env.update(env_extra)
    code = CHILD.replace("ROOT", repr(ROOT)).replace("ARGS", repr(args))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    for line in p.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    raise AssertionError((p.stderr or p.stdout)[-2000:])


CASES = [
    # rows, cols, typ, steps, gene, M  (cols = 128*M*C)
    (96, 1024, 2, 41, {}, 8),           # C=1: the ring wraps inside one CTA
    (96, 1024, 2, 41, {}, 4),           # C=2
    (200, 2048, 1, 64, {"a": -0.05}, 4),  # C=4, center-square init
    (130, 2048, 2, 37, {}, 16),         # C=1, M=16, ragged segments
    (64, 1024, 2, 30, {"dt": 100.0}, 8),  # blow-up: exact iteration and post-blow-up state
]


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,typ,steps,gene,m", CASES)
def test_rowring_bit_exact_vs_wavefront(rows, cols, typ, steps, gene, m):
    args = (rows, cols, typ, steps, gene)
    ref = run({"RDCNN_ROWRING": "0"}, args)
    # =2: any K=4 launch that cannot take the row-ring path fails the run
    got = run({"RDCNN_ROWRING": "2", "RDCNN_RR_M": str(m)}, args)
    assert got["rc"] in (0, 2) and ref["rc"] in (0, 2)  # RDCNN_OK / RDCNN_EBLOWUP
    assert got["checksum"] == ref["checksum"]
    assert (got["rc"], got["bad"]) == (ref["rc"], ref["bad"])
    if gene.get("dt") == 100.0:
        assert ref["bad"] > 0
