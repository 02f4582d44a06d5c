"""A/B of kernel paths chosen from the environment (one process per
variant): device Mcell-updates/s and the device checksum of the same run.

  --m 0,8,16          RDCNN_ROWRING=0 (wavefront) vs the row-ring kernel with M warps per CTA
  --variants "wf:RDCNN_RESIDENT=0;res2:RDCNN_RESIDENT=2,RDCNN_RES_K=2"
                      arbitrary named environments (the first is the checksum reference)

  python tools/rowring_ab.py --shapes 4096x4096,8192x8192 --iters 20000 --m 0,4,8,16
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]

CHILD = r"""
import json, sys, time
sys.path.insert(0, ROOT)
import paper_2102_10340_b200 as fhn
rows, cols, batch, iters, typ, mode, reps = ARGS
out = []
with fhn.Simulator(rows, cols, batch, levels=4, mode=mode, persistent=-1) as sim:
    sim.set_params(fhn.Gene(a=-0.05))
    sim.init(typ, 42)
    sim.advance(max(iters // 4, 4))
    best = 0.0
    for _ in range(reps):
        sim.advance(iters)
        ms = sim.elapsed_ms()
        best = max(best, rows * cols * batch * iters / ms / 1e3)
        out.append(round(rows * cols * batch * iters / ms / 1e3))
    cs = [int(x) for x in sim.checksums()]
    launches = sim.launch_count()
print("RESULT " + json.dumps({"mcells": out, "best": round(best), "checksum": "%016x" % cs[0],
                              "launches": launches}))
"""


def run(env_extra, rows, cols, batch, iters, typ, mode, reps):
    env = dict(os.environ)
    env.update(env_extra)
    code = CHILD.replace("ROOT", repr(ROOT)).replace("ARGS", repr((rows, cols, batch, iters, typ, mode, reps)))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    for line in p.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    return {"error": (p.stderr or p.stdout)[-600:]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096")
    ap.add_argument("--iters", type=int, default=20000)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--typ", type=int, default=1)
    ap.add_argument("--mode", default="strict")
    ap.add_argument("--m", default="0,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variants", default=None)
    a = ap.parse_args()
    if a.variants:
        vs = []
        for item in a.variants.split(";"):
            name, _, envs = item.partition(":")
            vs.append((name, dict(kv.split("=", 1) for kv in envs.split(",") if kv)))
        for shape in a.shapes.split(","):
            rows, cols = (int(x) for x in shape.split("x"))
            base = None
            for name, env in vs:
                r = run(env, rows, cols, a.batch, a.iters, a.typ, a.mode, a.reps)
                base = base or r
                print(f"{shape} {a.mode} {name}: {json.dumps(r)} same_as_first={r.get('checksum') == base.get('checksum')}",
                      flush=True)
        return
    for shape in a.shapes.split(","):
        rows, cols = (int(x) for x in shape.split("x"))
        base = None
        for m in (int(x) for x in a.m.split(",")):
            env = {"RDCNN_ROWRING": "0"} if m == 0 else {"RDCNN_ROWRING": "1", "RDCNN_RR_M": str(m)}
            r = run(env, rows, cols, a.batch, a.iters, a.typ, a.mode, a.reps)
            if m == 0:
                base = r
            same = base is not None and r.get("checksum") == base.get("checksum")
            tag = "wavefront" if m == 0 else f"rowring M={m}"
            print(f"{shape} batch={a.batch} {a.mode} {tag}: {json.dumps(r)} same_as_wavefront={same}", flush=True)


if __name__ == "__main__":
    main()
