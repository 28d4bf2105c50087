"""Static SASS instruction count of one walk step (the hot path of K1).

Traces the x2-unrolled step loop of walk_kernel<DV, Real, 0, true> in
libsddg.so with cuobjdump: from the loop head, taking the inner-box branch
(no exit, no bridge test) and the max-steps 'continue' branch, counting every
instruction on the way; the total over the two unrolled steps is halved.
Writes profiles/sass_walk_step.json (read by bench.py).

usage: python tools/sass_trace.py [--print]"""
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1310_3435_b200", "_lib", "libsddg.so")
KERNELS = {"fp64_ring": "_ZN4sddg11walk_kernelILi32EdLi0ELb1ELb0ELb0EEEvNS_8WalkArgsE",
           "fp32_shock": "_ZN4sddg11walk_kernelILi33EfLi0ELb1ELb0ELb0EEEvNS_8WalkArgsE"}
FP64 = ("DFMA", "DMUL", "DADD", "DSETP")


def trace(sass, fn):
    i = sass.index("Function : " + fn)
    j = sass.find("Function : ", i + 10)
    ins = []
    for line in sass[i:j if j > 0 else None].splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    idx = {o: k for k, (o, _) in enumerate(ins)}
    back = [(o, int(s.split()[-1], 16)) for o, s in ins
            if re.match(r"(@\S+ )?BRA (0x[0-9a-f]+)$", s) and int(s.split()[-1], 16) < o]
    head = max(back, key=lambda t: t[0] - t[1])[1]
    k, path = idx[head], []
    while len(path) < 4000:
        o, s = ins[k]
        path.append(s)
        m = re.match(r"(@!?U?P\d )?BRA (!?U?P\d, )?(0x[0-9a-f]+)$", s)
        if m:
            tgt = int(m.group(3), 16)
            if m.group(1) is None:
                k = idx[tgt]
            else:
                prev = [x for _, x in ins[max(0, k - 6):k]]
                box = m.group(2) is not None and sum(
                    ("SETP" in x) or ("PLOP3" in x) for x in prev) >= 3
                cont = any("ISETP.GE.U32" in x for x in prev[-3:]) and m.group(1).startswith("@!")
                k = idx[tgt] if (box or cont) else k + 1
        else:
            k += 1
        if k == idx[head]:
            break
    ops = Counter()
    for s in path:
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        ops[op.split(".")[0]] += 1
    return path, ops


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    out = {}
    for name, fn in KERNELS.items():
        path, ops = trace(sass, fn)
        steps = 2  # the loop body holds two steps
        out[name] = {"kernel": fn, "instructions_per_step": len(path) / steps,
                     "fp64_per_step": sum(ops[o] for o in FP64) / steps,
                     "opcodes_per_step": {k: v / steps for k, v in ops.most_common()}}
        if "--print" in sys.argv:
            print(name, out[name]["instructions_per_step"], out[name]["fp64_per_step"])
    json.dump(out, open(os.path.join(ROOT, "profiles", "sass_walk_step.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
