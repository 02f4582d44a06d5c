"""Instruction-class counts of one kernel's SASS (cuobjdump -sass), whole
function and the hottest loop (the largest backward-branch body).

  python tools/sass_classes.py <lib.so> <mangled-name-substring> [--dump out.sass]
"""
import argparse
import collections
import re
import subprocess

CLASSES = [
    ("fp32", r"^(FADD|FMUL|FFMA|FMNMX|FSETP|FSEL|FADD2|FMUL2|FFMA2|FMNMX3)\b"),
    ("shuffle", r"^SHFL\b"),
    ("smem", r"^(LDS|STS|LDSM)\b"),
    ("ldgsts/tma", r"^(LDGSTS|LDGDEPBAR|DEPBAR|UBLKCP|UTMALDG|SYNCS)\b"),
    ("global ld/st", r"^(LDG|STG|LD|ST|ATOM|RED|ATOMG)\b"),
    ("int/addr", r"^(IADD3|IADD|IMAD|LEA|SHF|LOP3|ISETP|IABS|IMNMX|SEL|MOV|PRMT|VIADD|VIMNMX|IMUL|I2F|F2I|POPC|FLO|BMSK|VIADDMNMX)\b"),
    ("uniform", r"^(U[A-Z0-9]+|R2UR|S2UR|VOTEU|ELECT)\b"),
    ("control", r"^(BRA|BRX|EXIT|RET|CALL|BSSY|BSYNC|WARPSYNC|BAR|NOP|YIELD|PLOP3|P2R|R2P|VOTE|WARPGROUP|ACQBULK|CCTL|MEMBAR|NANOSLEEP)\b"),
]


def classify(op):
    for name, pat in CLASSES:
        if re.match(pat, op):
            return name
    return "other"


def parse(text, sub):
    funcs = re.split(r"\n\s*Function : ", text)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if sub in name:
            return name, f
    raise SystemExit(f"no function matching {sub}")


def instrs(body):
    out = []
    for line in body.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", line)
        if m:
            out.append((int(m.group(1), 16), m.group(3), m.group(4), line.strip()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib")
    ap.add_argument("func")
    ap.add_argument("--dump", default=None)
    a = ap.parse_args()
    text = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    name, body = parse(text, a.func)
    ins = instrs(body)
    if a.dump:
        with open(a.dump, "w") as fh:
            fh.write(name + "\n" + "\n".join(i[3] for i in ins) + "\n")
    # largest backward branch = the hot loop
    best = None
    for addr, op, rest, _ in ins:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", rest)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                    best = (tgt, addr)
    def count(sel):
        c = collections.Counter(classify(op.split(".")[0]) for _, op, _, _ in sel)
        return c, len(sel)
    print(name)
    c, n = count(ins)
    print(f"whole function: {n} instructions")
    for k, v in sorted(c.items(), key=lambda kv: -kv[1]):
        print(f"  {k:14s} {v:6d}")
    if best:
        loop = [i for i in ins if best[0] <= i[0] <= best[1]]
        c, n = count(loop)
        print(f"hot loop [{best[0]:#x}, {best[1]:#x}]: {n} instructions")
        for k, v in sorted(c.items(), key=lambda kv: -kv[1]):
            print(f"  {k:14s} {v:6d} ({100.0 * v / n:.1f} %)")
        ops = collections.Counter(op for _, op, _, _ in loop)
        print("  top opcodes:", ", ".join(f"{o} {v}" for o, v in ops.most_common(25)))


if __name__ == "__main__":
    main()
