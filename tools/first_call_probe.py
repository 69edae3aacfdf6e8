"""Which part of a process's FIRST libvndf call waits for the GPU?  Each case
runs in a fresh interpreter: ~1 s of GPU sleep is queued on a stream, then the
first call is made on that stream; "pending" means the call returned while the
sleep was still running (no synchronisation).

    python tools/first_call_probe.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys, time
sys.path.insert(0, ROOTDIR)
import torch
import paper_2306_05044_b200 as vndf
torch.cuda.init()
dev = torch.device("cuda:0")
n = 1 << 20
o = vndf.empty_outputs(n, dev)
w = torch.empty(4 * n, dtype=torch.int32, device=dev)
c = torch.zeros(1, dtype=torch.int64, device=dev)
s = torch.cuda.Stream(dev)
vndf.lib()
PRESTMT
torch.cuda.synchronize()
with torch.cuda.stream(s):
    torch.cuda._sleep(2_000_000_000)
t0 = time.perf_counter()
CALLSTMT
dt = time.perf_counter() - t0
pending = not s.query()
s.synchronize()
print(f"{dt * 1e3:8.2f} ms  pending={pending}")
"""

CALLS = {
    "philox words (occupancy, no pool)": "vndf.vndf_philox4x32_10(3, 0, n, 0, w, stream=s)",
    "count fix-ups (occupancy, no pool)": "vndf.vndf_count_fixups_philox(3, 0, n, c, stream=s)",
    "heitz fused (no queue)": "vndf.vndf_sample_heitz2018_philox(3, 0, n, *o, stream=s)",
    "cap fused (pool + queue)": "vndf.vndf_sample_cap_philox(3, 0, n, *o, stream=s)",
}


PRE = {
    "first call": "pass",
    "after vndf_init": "vndf.vndf_init()",
    "after a words call": "vndf.vndf_philox4x32_10(3, 0, n, 0, w); torch.cuda.synchronize()",
}


def main():
    for env_name, pre in PRE.items():
        extra = {}
        for name, call in CALLS.items():
            env = dict(os.environ, **extra)
            r = subprocess.run([sys.executable, "-c", CASE.replace("ROOTDIR", repr(ROOT)).replace("CALLSTMT", call).replace("PRESTMT", pre)], env=env,
                               capture_output=True, text=True, timeout=300)
            out = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else ("FAILED " + r.stderr[-300:])
            print(f"{env_name:28s} {name:38s} {out}", flush=True)


if __name__ == "__main__":
    main()
