"""Instruction mix of every loop (backward branch) in one kernel's SASS.

    python tools/sass_loops.py [kernel-substring] [library]

Default: the Biot-Savart leaf-tile kernel k_tiles<0, 0> in the in-tree
library. Used to check, before spending GPU time, how many non-FP64
instructions each inner loop issues per pair block.
"""
import re
import subprocess
import sys
from collections import Counter

pat = sys.argv[1] if len(sys.argv) > 1 else "k_tilesILi0ELi0E"
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2401_07361_b200/lib/libspheresum_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
ins, on = [], False
for line in sass.split("\n"):
    if "Function : " in line:
        on = pat in line
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", line)
    if on and m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
print(f"{len(ins)} instructions")
at = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w*,\s*)?0x([0-9a-f]+)", t)
    if not m or int(m.group(1), 16) >= a or int(m.group(1), 16) not in at:
        continue
    body = ins[at[int(m.group(1), 16)] : i + 1]
    c = Counter(x.split()[1] if x.startswith("@") else x.split()[0] for _, x in body)
    dp = c["DFMA"] + c["DMUL"] + c["DADD"]
    lds = c["LDS.128"] + c["LDS"] + c["LDS.64"]
    print(f"loop {body[0][0]:#x}-{a:#x}: {len(body):4d} instr  fp64 {dp:3d}  mufu {c['MUFU.RCP64H']:2d}  "
          f"lds {lds:2d}  other {len(body) - dp - c['MUFU.RCP64H'] - lds}")
