"""Instruction mix of the main loop of a kernel in libvndf.so (static SASS).

python tools/sass_mix.py <substring of mangled name> [lib]
Counts instructions between the loop head (target of the backward branch that
closes the grid-stride loop) and that branch.
"""
import collections
import re
import subprocess
import sys

pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2306_05044_b200/libvndf.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    lines = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f)
    instrs = [(int(a, 16), t.strip()) for a, t in lines]
    # backward branches
    loops = []
    for addr, t in instrs:
        m = re.search(r"BRA(?:\.U)? (?:!?U?P\d+, )?(?:`\(\.L_x_\d+\) )?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < addr:
            loops.append((int(m.group(1), 16), addr))
    if not loops:
        print(name, "no loop")
        continue
    head, tail = max(loops, key=lambda p: p[1] - p[0])
    body = [t for a, t in instrs if head <= a <= tail]
    mix = collections.Counter()
    for t in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        mix[op.split(".")[0]] += 1
    print(name[:110])
    print(f"  loop 0x{head:x}-0x{tail:x}: {len(body)} instructions")
    print("  " + ", ".join(f"{k} {v}" for k, v in mix.most_common(40)))
