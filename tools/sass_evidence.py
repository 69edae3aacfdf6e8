"""SASS evidence per kernel of libvndf.so: static counts of the sm_100-specific
and pipe-relevant instructions (cuobjdump -sass).

python tools/sass_evidence.py r1 > profiles/r1/sass_evidence.txt
"""
import collections
import re
import subprocess
import sys

rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2306_05044_b200/libvndf.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
demangle = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function : (\S+)", out)),
                          capture_output=True, text=True).stdout.split("\n")
KEEP = re.compile(r"^(LDG\.\S*256\S*|STG\.\S*256|LDG\.\S*128\S*|STG\.\S*128|UBLKCP\S*|SYNCS\S*|ACQBULK\S*|PREEXIT\S*|"
                  r"MUFU\.\S+|IMAD\.WIDE\.U32|IMAD\.HI\.U32|DFMA|LDS\S*|ATOMS\S*|ATOMG\S*)$")
print(f"# SASS evidence ({rnd}): sm_100a-specific and pipe-relevant instructions per kernel of")
print("# libvndf.so (cuobjdump -sass; static counts, tools/sass_evidence.py).  LDG/STG ...256")
print("# = 256-bit global accesses (sm_100+; ELL2/EFL2 = L2 evict-last / evict-first hints);")
print("# UBLKCP + SYNCS = TMA bulk copy with an mbarrier; ACQBULK / PREEXIT =")
print("# griddepcontrol.wait / launch_dependents (programmatic dependent launch).")
print()
funcs = re.split(r"\n\s*Function : ", out)[1:]
for k, f in enumerate(funcs):
    name = demangle[k] if k < len(demangle) else f.split("\n", 1)[0]
    name = re.sub(r"\(anonymous namespace\)::", "", name).split("(")[0]
    c = collections.Counter()
    for op in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", f):
        if KEEP.match(op):
            c[op] += 1
    if c:
        print(name)
        print("    " + ", ".join(f"{op} {n}" for op, n in sorted(c.items(), key=lambda kv: (-kv[1], kv[0]))))
