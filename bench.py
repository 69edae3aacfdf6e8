#!/usr/bin/env python
"""bench.py -- throughput of GGX VNDF spherical-cap sampling on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the whole hot path over one batch of BASELINE.json
configs[3] (config 4, the largest single-GPU configuration: 2^30 samples,
in-kernel Philox4x32-10 inputs with key = seed 3 and counter = sample index,
wi uniform on the upper hemisphere, alpha_x, alpha_y log-uniform [0.01, 1],
u1, u2; output h + pdf, 16 B per sample), i.e. ONE call of
vndf_sample_cap_philox: input generation, stretch, spherical cap, half
vector, unstretch, Eq. 1 pdf, float64 fix-up of the flagged samples (the fused
kernel plus the fix-up kernel).  The 17.2 GB of outputs per step exceed the
126 MB L2 many times over, so no flush is needed.  Under torchrun each rank
processes its own batch (global indices rank * 2^30 ...): weak scaling, no
data-path collective (DESIGN.md s.7).

Prints ONE JSON line on rank 0 (all other output goes to stderr).  `value` is
whole-job Gsamples/s timed with CUDA events on the launching stream, max over
ranks; `e2e` is the same metric through the blocking host-buffer entry point
vndf_sample_cap_philox_host (pinned host outputs written across the link inside
the timed region); `roofline` is the fused kernel's issue roofline; `c3`, `c5`,
`c1`, `c2` are the streamed configurations (the HBM roofline run is c3);
`cpu_baseline` is the float64 oracle on this box's cores (bounded samples), and
its leg also checks the headline's outputs at sampled indices against it.
`--impl reference` times the oracle itself (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Gsamples/s of GGX VNDF spherical-cap sampling; % HBM/FP32 roofline; vs Heitz18"
UNIT = "Gsamples/s"
WORKLOAD_CID = 4
C4_SEED = 3
FALLBACK_HBM_GBS = 6650.0                   # B200_PROFILING.md fallback, if MEASURED_PEAKS.json is absent
SMS, SMSPS_PER_SM, SM_MAX_MHZ = 148, 4, 1965.0
TOL_H, TOL_PDF = 2e-5, 1e-4                 # BASELINE.json north_star parity contract


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-variants", action="store_true", help="skip the streamed-config and NEXT side runs")
    p.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard_first_index(rank: int, n: int) -> int:
    """Weak scaling: rank r owns global samples [r n, (r + 1) n).  The inputs are
    counter-based, so a sample's value depends only on its global index."""
    return rank * n


def reduce_max(value: float, world: int, device=None) -> float:
    """Max over ranks (timings): an all-reduce MAX when world > 1."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _measured():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def peaks():
    mp = _measured()
    if "hbm_gbs" in mp:
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", mp
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


def _profiled(key: str):
    """A per-kernel figure from the committed ncu captures (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """Polls NVML SM clock and clock-event reasons during the timed region."""

    BAD = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons, self.power = [], set(), []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = self._handle(nv, index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    @staticmethod
    def _handle(nv, index):
        """NVML handle of CUDA device `index`, matched by PCI bus id (NVML and CUDA
        enumerate devices in different orders, and CUDA_VISIBLE_DEVICES remaps)."""
        try:
            import torch
            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(index)

    def _poll(self):
        nv = self._nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            try:
                self.power.append(nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0)
            except Exception:
                pass
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                     nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                     nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                     nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                     nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake_slowdown"}
            for bit, nm in names.items():
                if r & bit:
                    self.reasons.add(nm)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._poll()
            time.sleep(self.period)

    def start(self):
        if self._nv is None:
            return
        self._poll()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        if self._nv is None:
            return
        self._stop.set()
        self._t.join()
        self._poll()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        s = sorted(self.samples)
        out = {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
               "n_samples": len(s)}
        if self.power:
            out["power_w_max"] = round(max(self.power), 1)
        return out


# ------------------------------------------------------------ timed loops ---
def time_launches(torch, fn, steps: int, warmup: int, stream, per_step: bool = True):
    """W untimed warm-up launches, then `steps` launches bracketed by events on
    `stream`.  Returns (total_ms, per_launch_ms list).  per_step=False records
    only the two bracketing events (an event between two launches stops the
    next launch from overlapping the previous one's tail)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range((steps if per_step else 1) + 1)]
    ev[0].record(stream)
    for k in range(steps):
        fn()
        if per_step:
            ev[k + 1].record(stream)
    if not per_step:
        ev[1].record(stream)
    torch.cuda.synchronize()
    if per_step:
        per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
        return ev[0].elapsed_time(ev[steps]), per
    total = ev[0].elapsed_time(ev[1])
    return total, [total / steps] * steps


# ------------------------------------------------------------- rooflines ---
def roofline(bytes_per_launch: float, launch_ms: float, kernel_key: str):
    """HBM roofline of a streamed kernel: algorithmic bytes / launch time against
    the measured copy bandwidth (MEASURED_PEAKS.json)."""
    peak, src, _ = peaks()
    achieved = bytes_per_launch / (launch_ms * 1e-3) / 1e9
    probe = _profiled("pattern_probe_7r4w_2e24_gbs")
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": _profiled(kernel_key),
            "peak_source": src, "kernel": kernel_key,
            "algorithmic_bytes_per_launch": int(bytes_per_launch),
            # context only: the HGX figure (B200_PROFILING.md) and the same plane
            # pattern with no arithmetic (tools/bw_probe.cu)
            "frac_of_spec_7700": round(achieved / 7700.0, 4),
            "frac_of_pattern_probe": round(achieved / probe, 4) if probe else None}


def issue_roofline(gsamples_s: float, key: str, n_per_launch: int = None, launch_ms: float = None):
    """Issue roofline of a compute-bound fused kernel (DESIGN.md s.6.4): each of
    the 4 SMSPs of the 148 SMs issues at most one warp-instruction per clock at
    the 1965 MHz maximum SM clock (the guide's unit counts and clocks), so the
    peak is 592 x 1.965 G warp-inst/s; achieved = the kernel's ncu-counted
    warp-instructions per sample x samples / time.  frac is the share of issue
    slots the kernel fills; peak / inst gives the Gsamples/s bound."""
    inst = _profiled(key)
    if not inst:
        return None
    f = SM_MAX_MHZ * 1e6
    peak = SMS * SMSPS_PER_SM * f / 1e9
    achieved = gsamples_s * inst
    out = {"bound": "alu", "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": "Gwarp-inst/s",
           "frac": round(achieved / peak, 4), "traffic": None,
           "warp_inst_per_sample": inst, "gsamples_s_bound": round(peak / inst, 2),
           "model": "592 SMSPs x 1 warp-inst/clk x 1965 MHz; ncu warp-inst/sample (DESIGN.md s.6.4)"}
    # the FMA datapath: IMAD.WIDE.U32 (Philox) holds it ~4.3 clk per warp-instruction
    # and does not overlap with FP32 FFMA/FMUL on B200 (tools/mix_probe.cu), so the
    # sum of the measured per-instruction costs bounds the kernel (DESIGN.md s.6.5)
    cyc = _profiled(key.replace("warp_inst_per_sample", "fma_pipe_cycles_per_warp_sample"))
    if cyc:
        bound = SMS * SMSPS_PER_SM * f * 32 / cyc / 1e9
        out["fma_pipe"] = {"cycles_per_warp_sample": cyc, "gsamples_s_bound": round(bound, 2),
                           "frac": round(gsamples_s / bound, 4),
                           "model": "measured clk per IMAD.WIDE / FFMA 3-reg / other FP32 / IMAD x ncu counts "
                                    "(DESIGN.md s.6.5)"}
    return out


# ----------------------------------------------------------------- oracle ---
def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _rate(fn, n, reps, budget_s=None):
    """Median samples/s of `reps` runs of fn() (or as many as fit in budget_s)."""
    ts = []
    t_end = time.perf_counter() + (budget_s or 1e9)
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if budget_s and time.perf_counter() > t_end and len(ts) >= 3:
            break
    ts.sort()
    return n / ts[len(ts) // 2] / 1e9, len(ts)


def cpu_baseline(check=None, c1_planes=None, c3_planes=None, budget_s: float = 10.0, log2_sub: int = 24):
    """The float64 oracle, as it stands, on this box's host cores (SURVEY 8(d):
    1 thread and T threads): the headline's config-4 recipe on bounded
    sub-ranges, plus config 1 (median of 100, the paper's methodology)
    and a 2^24 sub-range of config 3.  `check` = (indices, h[3, m], pdf[m]) of
    the GPU headline run: compared with the oracle at those indices."""
    import numpy as np
    import oracle
    oracle.build()
    T = oracle.default_threads()
    m = 1 << min(22, log2_sub)
    idx = np.arange(m, dtype=np.uint64)
    # headline value: config 4, 2^22 indices, T threads, repeated within the budget
    done, t0 = 0, time.perf_counter()
    while True:
        oracle.batch_sample_philox(oracle.CAP, C4_SEED, idx, threads=T)
        done += m
        if time.perf_counter() - t0 >= budget_s * 0.4:
            break
    dt = time.perf_counter() - t0
    out = {"value": round(done / dt / 1e9, 5), "unit": UNIT, "cores": T, "kind": "oracle",
           "sample": f"config-4 indices [0, 2^22) x {done // m} in {dt:.1f} s, {T} threads",
           "cpu_model": _cpu_model()}
    sub = {}
    ns, n1 = 1 << log2_sub, 1 << (log2_sub - 4)
    i24 = np.arange(ns, dtype=np.uint64)
    r1, k1 = _rate(lambda: oracle.batch_sample_philox(oracle.CAP, C4_SEED, i24[:n1], threads=1), n1, 5)
    rT, kT = _rate(lambda: oracle.batch_sample_philox(oracle.CAP, C4_SEED, i24, threads=T), ns, 5)
    sub["c4_2e24"] = {"T_threads": round(rT, 5), "1_thread": round(r1, 5), "runs": [kT, k1],
                      "note": "T: median of 5 on 2^24; 1: on 2^20"}
    if c1_planes is not None:
        n1p = c1_planes[0].size
        rT, kT = _rate(lambda: oracle.batch_sample(oracle.CAP, *c1_planes, pdf=True, threads=T), n1p, 100)
        r1, k1 = _rate(lambda: oracle.batch_sample(oracle.CAP, *c1_planes, pdf=True, threads=1), n1p, 100,
                       budget_s=2.0)
        sub["c1_2e16"] = {"T_threads": round(rT, 5), "1_thread": round(r1, 5), "runs": [kT, k1],
                          "note": "median of 100 (1 thread: within 2 s)"}
    if c3_planes is not None:
        rT, kT = _rate(lambda: oracle.batch_sample(oracle.CAP, *c3_planes, pdf=False, threads=T),
                       c3_planes[0].size, 5)
        one = [p[:n1] for p in c3_planes]
        r1, k1 = _rate(lambda: oracle.batch_sample(oracle.CAP, *one, pdf=False, threads=1), one[0].size, 5)
        sub["c3_2e24"] = {"T_threads": round(rT, 5), "1_thread": round(r1, 5), "runs": [kT, k1],
                          "note": "T: median of 5 on 2^24; 1: on 2^20"}
    out["subranges"] = sub
    if check is not None:
        ci, ch, cp = check
        h_ref, p_ref, _ = oracle.batch_sample_philox(oracle.CAP, C4_SEED, ci, threads=T)
        dh = np.abs(ch.astype(np.float64) - h_ref).max(axis=0)
        dp = np.abs(cp.astype(np.float64) - p_ref) / p_ref
        out["parity_vs_gpu"] = {"samples": int(ci.size), "max_abs_dh": float(dh.max()),
                                "max_rel_dpdf": float(dp.max()), "over_tol": int(((dh > TOL_H) | (dp > TOL_PDF)).sum()),
                                "tol": [TOL_H, TOL_PDF]}
    return out


# ----------------------------------------------------------------- ours ---
def _git_sha():
    """The commit of the sources: from git where there is a checkout, else from
    the build_info.json that build() wrote beside the library, if it describes
    these very sources (same source hash)."""
    try:
        sha = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if sha:
            return sha
    except Exception:
        pass
    try:
        from paper_2306_05044_b200 import _build
        with open(_build.BUILD_INFO) as f:
            info = json.load(f)
        if info.get("libvndf_source_sha256") == _build.source_hash():
            return info["git"] + ("-dirty" if info.get("git_dirty") else "")
    except Exception:
        pass
    return None


def _sha256(tensors, limit):
    h = hashlib.sha256()
    for t in tensors:
        h.update(t[:limit].cpu().numpy().tobytes())
    return h.hexdigest()


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    import __graft_entry__
    __graft_entry__.build()
    import paper_2306_05044_b200 as vndf
    from paper_2306_05044_b200 import _build
    import synth

    cfg = synth.CONFIGS[WORKLOAD_CID]
    n = cfg.n
    first = shard_first_index(rank, n)
    stream = torch.cuda.current_stream(dev)
    vndf.vndf_init(dev.index)
    out = vndf.empty_outputs(n, dev, pdf=True)
    torch.cuda.synchronize()

    def step():
        vndf.vndf_sample_cap_philox(C4_SEED, first, n, *out, stream=stream)

    barrier = (lambda: dist.barrier()) if world > 1 else None
    clocks = ClockSampler(dev.index)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    clocks.start()
    total_ms, _ = time_launches(torch, step, args.steps, 0, stream, per_step=False)
    clocks.stop()
    if barrier:
        barrier()
    total_ms = reduce_max(total_ms, world, dev)
    ms_per_step = total_ms / args.steps
    value = world * n * args.steps / (total_ms * 1e-3) / 1e9

    # fix-up count of the workload (diagnostic kernel, outside the timed region)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    vndf.vndf_count_fixups_philox(C4_SEED, first, n, cnt, stream=stream)
    # outputs at sampled indices for the oracle check (cpu_baseline leg)
    g = torch.Generator().manual_seed(1234)
    ci = torch.cat([torch.randint(0, n, (1 << 18,), generator=g), torch.arange(0, 4096),
                    torch.arange(n - 4096, n)]).to(dev)
    check_h = torch.stack([t[ci] for t in out[:3]]).cpu().numpy()
    check_p = out[3][ci].cpu().numpy()
    check_i = (ci.cpu().numpy().astype(np.uint64) + np.uint64(first))
    out_sha = _sha256(out, 1 << 24)
    torch.cuda.synchronize()
    fixups = int(cnt.item())
    del out
    torch.cuda.empty_cache()

    rl = issue_roofline(value / world, "cap_philox_c4_warp_inst_per_sample")
    if rl is not None:
        rl["traffic"] = _profiled("cap_philox_c4_dram_bytes")
        rl["algorithmic_bytes_per_launch"] = 16 * n
        rl["pipes_ncu"] = _profiled("cap_philox_c4_pipes")
        rl["kernel"] = "philox_kernel<cap> + philox_fixup_kernel (the whole step)"

    # ---- end to end: the host-buffer entry point, pinned host outputs ----
    e2e = None
    if not args.no_e2e:
        # one rank: the whole 2^30-sample step (17.2 GB of pinned host planes);
        # several ranks on one node share its host memory, so each writes a
        # quarter of its batch (the rate, not the batch, is the metric)
        ne = n if world == 1 else n >> 2
        hout = [torch.empty(ne, dtype=torch.float32, pin_memory=True) for _ in range(4)]
        vndf.vndf_sample_cap_philox_host(C4_SEED, first, ne, *hout)           # warm-up
        e2e_steps = 3
        if barrier:
            barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            vndf.vndf_sample_cap_philox_host(C4_SEED, first, ne, *hout)
        e2e_s = reduce_max(time.perf_counter() - t0, world, dev)
        same = bool(hashlib.sha256(b"".join(t[: 1 << 24].numpy().tobytes() for t in hout)).hexdigest() == out_sha)
        # the host link's own device -> pinned host rate (a plain 1 GiB copy): the e2e ceiling
        src = torch.empty(1 << 28, dtype=torch.float32, device=dev)
        dst = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
        dst.copy_(src)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(3):
            dst.copy_(src)
        torch.cuda.synchronize()
        link_peak = 3 * (1 << 30) / (time.perf_counter() - t1) / 1e9
        del src, dst
        link = 16 * ne * e2e_steps / e2e_s / 1e9
        e2e = {"value": round(world * ne * e2e_steps / e2e_s / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 16 * ne, "samples_per_rank_per_step": ne,
               "api": "vndf_sample_cap_philox_host (2 Mi-sample chunks, DMA into pinned host planes)",
               "steps": e2e_steps, "bit_identical_to_device": same,
               "link_gb_s": round(link, 2), "link_d2h_copy_gb_s": round(link_peak, 2),
               "frac_of_link": round(link / link_peak, 4)}
        del hout

    result = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (in-kernel Philox4x32-10, config-4 recipe)",
        "config": {"workload": f"config 4: {cfg.label}", "samples_per_gpu_per_step": n,
                   "kernel": "vndf_sample_cap_philox", "parallelism": f"independent shards x{world}",
                   "l2": "17.2 GB written per step >> 126 MB L2, no flush"},
        "roofline": rl,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "gpu_launches": 2 * args.steps,
        "fixups": {"count": fixups, "rate": round(fixups / n, 7)},
        "build": {"git": _git_sha(), "libvndf_source_sha256": _build.source_hash()[:16]},
        "outputs_sha256_first_2e24": out_sha[:16],
    }

    if world == 1 and not args.no_variants:
        result.update(side_runs(torch, vndf, synth, dev, stream, value))
    if rank == 0 and world == 1 and not args.no_cpu:
        c1 = synth.CONFIGS[1]
        c1p = [v.cpu().numpy() for v in synth.fill(c1.recipe, c1.seed, c1.n, device=dev).values()]
        c3 = synth.CONFIGS[3]
        x3 = synth.fill(c3.recipe, c3.seed, 1 << 24, device=dev)
        c3p = [x3[k].cpu().numpy() for k in synth.PLANES]
        del x3
        cb = cpu_baseline(check=(check_i, check_h, check_p), c1_planes=c1p, c3_planes=c3p)
        result["parity"] = cb.pop("parity_vs_gpu")
        result["cpu_baseline"] = cb
        result["chi2"] = chi2_pvalues(torch, vndf, synth, dev)
        if "_c5_kept" in result:
            c5_over_tolerance(result["c5"]["robustness"], result["_c5_kept"])
    elif rank == 0:
        result["cpu_baseline"] = None
    result.pop("_c5_kept", None)
    if rank == 0:
        print(json.dumps(ordered(result), separators=(",", ":")), flush=True)
    if world > 1:
        dist.destroy_process_group()


CHI2_PAIRS = [(0, 0, 1, 1), (0, 0, .5, .5), (45, 0, .2, .2), (80, 30, .5, .5),
              (70, 20, .05, .3), (85, 60, .3, .05), (45, 0, .01, .01), (60, 135, 1, .1)]


def chi2_pvalues(torch, vndf, synth, dev, n: int = 1 << 21, seed: int = 1000):
    """BJ config 2's distribution check in the bench run: 64 x 64 (theta, phi)
    histograms of h from the cap and Heitz kernels, 2^21 samples for each of the
    eight fixed (wi, alpha) pairs, Pearson chi-square against the oracle's Eq. 1
    quadrature masses (reading R14; tests/test_distribution_gpu.py
    holds the 3-seed gate)."""
    import numpy as np
    from oracle import stats
    out = {"n_per_pair": n, "seed": seed, "pairs_theta_phi_ax_ay": CHI2_PAIRS, "cap_p": [], "heitz_p": []}
    for t, p, ax, ay in CHI2_PAIRS:
        tr, pr = np.radians(t), np.radians(p)
        wi = np.array([np.sin(tr) * np.cos(pr), np.sin(tr) * np.sin(pr), np.cos(tr)], dtype=np.float32)
        masses = stats.bin_masses(wi.astype(np.float64), ax, ay)
        x = synth.fill(0, seed, n, device=dev, fixed=[wi[0], wi[1], wi[2], ax, ay])
        ins = [x[k] for k in synth.PLANES]
        o = vndf.empty_outputs(n, dev)
        for name, fn in (("cap_p", vndf.vndf_sample_cap_pdf), ("heitz_p", vndf.vndf_sample_heitz2018)):
            fn(*ins, *o)
            torch.cuda.synchronize()
            h = np.stack([q.cpu().numpy() for q in o[:3]]).astype(np.float64)
            _, _, pv = stats.pearson(stats.histogram(h), masses)
            out[name].append(float(f"{pv:.3g}"))
    out["cap_min_p"], out["heitz_min_p"] = min(out["cap_p"]), min(out["heitz_p"])
    return out


CONTRACT_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                 "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches")


# The driver keeps the contract keys of the line (parsed) and the last ~3 KB of
# stdout: the per-config objects that matter go last, the summary at the very end.
TAIL_KEYS = ("fixups", "c1", "c2", "c5", "c5_fused", "heitz_c4", "c3", "parity")


def summary(r):
    """The per-config headline numbers in one short object, the last key of the
    line (a record that keeps only the tail of stdout keeps them)."""
    def g(*path):
        v = r
        for k in path:
            if not isinstance(v, dict) or k not in v:
                return None
            v = v[k]
        return v
    return {"c4_gsamples_s": r.get("value"), "c4_frac_issue": g("roofline", "frac"),
            "c4_frac_fma_pipe": g("roofline", "fma_pipe", "frac"), "c4_t_heitz_over_t_cap": g("heitz_c4", "t_heitz_over_t_cap"),
            "c3_gb_s": g("c3", "gb_s"), "c3_frac_hbm": g("c3", "frac_hbm"), "c3_t_heitz_over_t_cap": g("c3", "t_heitz_over_t_cap"),
            "c5_t_heitz_over_t_cap": g("c5", "t_heitz_over_t_cap"),
            "c5_fused_t_heitz_over_t_cap": g("c5_fused", "t_heitz_over_t_cap"),
            "c1_cap_us": g("c1", "cap_us"), "c1_t_heitz_over_t_cap": g("c1", "t_heitz_over_t_cap"),
            "c2_frac_hbm": g("c2", "frac_hbm"),
            "sampler_only_t_heitz_over_t_cap": g("next", "microbench_t_heitz_over_t_cap"),
            "parity_over_tol": g("parity", "over_tol"), "chi2_cap_min_p": g("chi2", "cap_min_p"),
            "cpu_oracle_gsamples_s": g("cpu_baseline", "value")}


def ordered(r):
    out = {k: r[k] for k in CONTRACT_KEYS if k in r}
    out.update({k: v for k, v in r.items() if k not in out and k not in TAIL_KEYS})
    out.update({k: r[k] for k in TAIL_KEYS if k in r})
    out["summary"] = summary(r)
    return out


def c5_robustness(torch, vndf, ins, out, n, dev, m: int = 1 << 16):
    """SURVEY 8(d) config 5 robustness, cap and Heitz on the same 2^26 edge-mix
    inputs: NaN count and invariant violations on EVERY sample, on the device
    (|h| = 1 within 1e-5, s h.z >= 0 and wi.h >= 0 within 1e-6, reading R4); the
    outputs at m sampled indices are kept for the cpu_baseline leg, which counts
    those over the 2e-5 / 1e-4 contract against the float64 oracle."""
    wx, wy, wz = ins[0], ins[1], ins[2]
    s = torch.where(wz < 0, -1.0, 1.0)
    g = torch.Generator().manual_seed(55)
    idx = torch.randint(0, n, (m,), generator=g).to(dev)
    res, kept = {}, {"inputs": [t[idx].cpu().numpy() for t in ins]}
    for name, fn in (("cap", vndf.vndf_sample_cap_pdf), ("heitz", vndf.vndf_sample_heitz2018)):
        fn(*ins, *out)
        hx, hy, hz, pd = out
        nan = int((~torch.isfinite(hx) | ~torch.isfinite(hy) | ~torch.isfinite(hz) | ~torch.isfinite(pd)).sum())
        nrm = (hx.double() ** 2 + hy.double() ** 2 + hz.double() ** 2 - 1.0).abs()
        inv = int(((nrm > 1e-5) | (s * hz < -1e-6) | (wx * hx + wy * hy + wz * hz < -1e-6)).sum())
        res[name] = {"nan": nan, "invariant_violations": inv}
        kept[name] = [o[idx].cpu().numpy() for o in out]
    return res, kept


def c5_over_tolerance(robust, kept):
    """The cpu_baseline leg's half of c5_robustness: sampled outputs against the oracle."""
    import numpy as np
    import oracle
    for name, method in (("cap", oracle.CAP), ("heitz", oracle.HEITZ)):
        hr, pr, _ = oracle.batch_sample(method, *kept["inputs"], pdf=True)
        hg = np.stack(kept[name][:3]).astype(np.float64)
        pg = kept[name][3].astype(np.float64)
        over = (np.abs(hg - hr).max(axis=0) > TOL_H) | (np.abs(pg - pr) / pr > TOL_PDF)
        robust[name]["over_tolerance"] = int(over.sum())
        robust[name]["of_sampled"] = int(pg.size)


def side_runs(torch, vndf, synth, dev, stream, c4_value):
    """The other configurations and the Heitz-2018 baseline on identical inputs
    (3 warm-up + 20 timed launches each; cap and Heitz alternated 3 times,
    medians), compact: c4 Heitz ratio, c3 (HBM
    roofline run), c5 (edge mix), c1 (latency), c2, then the NEXT rows."""
    res = {}
    reps, warm = 20, 3

    def timed(fn, r=reps):
        total, _ = time_launches(torch, fn, r, warm, stream, per_step=False)
        return total / r

    def timed_pair(fa, fb, rounds=3):
        """Cap and Heitz alternated over a few rounds, median of each: drift of
        the device state (the board's power limit, profiles/r2/power_state_probe_r2.txt)
        then hits both alike."""
        ta, tb = [], []
        for _ in range(rounds):
            ta.append(timed(fa))
            tb.append(timed(fb))
        return sorted(ta)[rounds // 2], sorted(tb)[rounds // 2]

    def gs(n, ms):
        return round(n / ms / 1e6, 2)

    c4 = synth.CONFIGS[4]
    o4 = vndf.empty_outputs(c4.n, dev)
    t_h4 = timed(lambda: vndf.vndf_sample_heitz2018_philox(C4_SEED, 0, c4.n, *o4, stream=stream), 10)
    hz = gs(c4.n, t_h4)
    res["heitz_c4"] = {"gsamples_s": hz, "t_heitz_over_t_cap": round(c4_value / hz, 4),
                       "roofline": issue_roofline(hz, "heitz_philox_c4_warp_inst_per_sample")}
    del o4
    torch.cuda.empty_cache()

    # config 5's edge mix generated in-kernel (fused): grazing and below-horizon
    # incidence in the compute-bound variant, cap vs Heitz on identical inputs
    c5 = synth.CONFIGS[5]
    o5 = vndf.empty_outputs(c5.n, dev)
    t_ce, t_he = timed_pair(lambda: vndf.vndf_sample_cap_philox_edge(c5.seed, 0, c5.n, *o5, stream=stream),
                            lambda: vndf.vndf_sample_heitz2018_philox_edge(c5.seed, 0, c5.n, *o5, stream=stream))
    res["c5_fused"] = {"gsamples_s": gs(c5.n, t_ce), "heitz_gsamples_s": gs(c5.n, t_he),
                       "t_heitz_over_t_cap": round(t_he / t_ce, 4)}
    del o5
    torch.cuda.empty_cache()

    # config 3: 2^28 streamed, h only -- the HBM roofline run
    c3 = synth.CONFIGS[3]
    x3 = synth.fill(c3.recipe, c3.seed, c3.n, device=dev)
    o3 = vndf.empty_outputs(c3.n, dev, pdf=False)
    ins3 = [x3[k] for k in synth.PLANES]
    t_cap3, t_hz3 = timed_pair(lambda: vndf.vndf_sample_cap(*ins3, *o3, stream=stream),
                               lambda: vndf.vndf_sample_heitz2018(*ins3, *o3, None, stream=stream))
    rl3 = roofline(40 * c3.n, t_cap3, "cap_c3")
    res["c3"] = {"gsamples_s": gs(c3.n, t_cap3), "ms": round(t_cap3, 4), "gb_s": rl3["achieved"],
                 "frac_hbm": rl3["frac"], "t_heitz_over_t_cap": round(t_hz3 / t_cap3, 4), "roofline": rl3,
                 "inputs_sha256_first_2e20": _sha256(ins3, 1 << 20)[:16]}
    # config 3 end to end: pinned host planes in (28 B) and out (12 B), zero-copy
    hin3 = [t.cpu().pin_memory() for t in ins3]
    del x3, o3, ins3
    torch.cuda.empty_cache()
    hout3 = [torch.empty(c3.n, dtype=torch.float32, pin_memory=True) for _ in range(3)]
    vndf.vndf_sample_cap_pdf_host(*hin3, *hout3, None)
    t0 = time.perf_counter()
    for _ in range(3):
        vndf.vndf_sample_cap_pdf_host(*hin3, *hout3, None)
    e3 = (time.perf_counter() - t0) / 3
    res["c3"]["e2e"] = {"gsamples_s": round(c3.n / e3 / 1e9, 4), "link_gb_s": round(40 * c3.n / e3 / 1e9, 2),
                        "api": "vndf_sample_cap_pdf_host (pdf NULL, zero-copy)"}
    del hin3, hout3
    torch.cuda.empty_cache()

    # config 5: 2^26 edge mix, h + pdf (flip frame and the native frame)
    c5 = synth.CONFIGS[5]
    x5 = synth.fill(c5.recipe, c5.seed, c5.n, device=dev)
    o5 = vndf.empty_outputs(c5.n, dev)
    ins5 = [x5[k] for k in synth.PLANES]
    t_cap5, t_hz5 = timed_pair(lambda: vndf.vndf_sample_cap_pdf(*ins5, *o5, stream=stream),
                               lambda: vndf.vndf_sample_heitz2018(*ins5, *o5, stream=stream))
    t_nat5 = timed(lambda: vndf.vndf_sample_cap_pdf_native(*ins5, *o5, stream=stream))
    res["c5"] = {"gsamples_s": gs(c5.n, t_cap5), "t_heitz_over_t_cap": round(t_hz5 / t_cap5, 4),
                 "frac_hbm": roofline(44 * c5.n, t_cap5, "cap_pdf_c5")["frac"],
                 "native_gsamples_s": gs(c5.n, t_nat5)}
    res["c5"]["robustness"], res["_c5_kept"] = c5_robustness(torch, vndf, ins5, o5, c5.n, dev)
    del x5, o5, ins5

    # config 1: 2^16 samples, L2-resident and launch-bound (us per
    # launch): 50 launches in one CUDA graph, replayed
    c1 = synth.CONFIGS[1]
    x1 = synth.fill(c1.recipe, c1.seed, c1.n, device=dev)
    o1 = vndf.empty_outputs(c1.n, dev)
    ins1 = [x1[k] for k in synth.PLANES]
    vndf.vndf_sample_cap_pdf(*ins1, *o1)
    vndf.vndf_sample_heitz2018(*ins1, *o1)
    torch.cuda.synchronize()
    c1res = {}
    for name, fn in (("cap_us", vndf.vndf_sample_cap_pdf), ("heitz_us", vndf.vndf_sample_heitz2018)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(50):
                fn(*ins1, *o1)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        per = []
        for _ in range(5):  # median of 5 x (10 replays of 50 launches)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(10):
                g.replay()
            ev1.record()
            torch.cuda.synchronize()
            per.append(ev0.elapsed_time(ev1) * 1e3 / 500)
        c1res[name] = round(sorted(per)[2], 3)
    c1res["t_heitz_over_t_cap"] = round(c1res["heitz_us"] / c1res["cap_us"], 4)
    res["c1"] = c1res
    del x1, o1, ins1

    # config 2: 2^24, h + pdf
    c2 = synth.CONFIGS[2]
    x2 = synth.fill(c2.recipe, c2.seed, c2.n, device=dev)
    o2 = vndf.empty_outputs(c2.n, dev)
    ins2 = [x2[k] for k in synth.PLANES]
    t_cap2, t_hz2 = timed_pair(lambda: vndf.vndf_sample_cap_pdf(*ins2, *o2, stream=stream),
                               lambda: vndf.vndf_sample_heitz2018(*ins2, *o2, stream=stream))
    res["c2"] = {"gsamples_s": gs(c2.n, t_cap2), "frac_hbm": roofline(44 * c2.n, t_cap2, "cap_pdf_c2")["frac"],
                 "t_heitz_over_t_cap": round(t_hz2 / t_cap2, 4)}

    nxt = {}
    # NEXT-1: sampler-only microbenchmark in the paper's methodology:
    # 64 Listing-1 calls per lane, median of 100 dispatches
    lanes, iters = 148 * 2048 * 16, 64
    ck = torch.empty(lanes, dtype=torch.float32, device=dev)
    mb = {}
    for method, name in ((0, "cap"), (1, "heitz"), (2, "cap_literal")):
        _, per = time_launches(torch, lambda: vndf.vndf_microbench(method, 5, lanes, iters, ck, stream=stream),
                               100, 5, stream)
        mb[name] = sorted(per)[len(per) // 2]
    nxt["microbench_t_heitz_over_t_cap"] = round(mb["heitz"] / mb["cap"], 4)
    nxt["microbench_t_heitz_over_t_cap_literal"] = round(mb["heitz"] / mb["cap_literal"], 4)
    nxt["microbench_cap_gsamples_s"] = gs(lanes * iters, mb["cap"])
    del ck
    # NEXT-2: reflection on the config-2 inputs; fused on config-4 inputs
    ro = [torch.empty(c2.n, dtype=torch.float32, device=dev) for _ in range(5)]
    t_r = timed(lambda: vndf.vndf_sample_cap_reflect(*ins2, *ro, stream=stream))
    nxt["reflect_c2_frac_hbm"] = roofline(48 * c2.n, t_r, "cap_reflect_c2")["frac"]
    # NEXT-4: Eq. 1 at caller-provided h
    t_p = timed(lambda: vndf.vndf_pdf(*ro[:3], *ins2[:5], ro[3], stream=stream))
    nxt["pdf_c2_frac_hbm"] = roofline(36 * c2.n, t_p, "pdf_c2")["frac"]
    del ro, x2, o2, ins2
    nr = 1 << 28
    orf = [torch.empty(nr, dtype=torch.float32, device=dev) for _ in range(5)]
    t_rc = timed(lambda: vndf.vndf_sample_cap_reflect_philox(C4_SEED, 0, nr, *orf, stream=stream))
    t_rh = timed(lambda: vndf.vndf_sample_heitz2018_reflect_philox(C4_SEED, 0, nr, *orf, stream=stream))
    nxt["reflect_philox_gsamples_s"] = gs(nr, t_rc)
    nxt["reflect_philox_t_heitz_over_t_cap"] = round(t_rh / t_rc, 4)
    del orf
    # NEXT-2: Eq. 19 white-furnace estimator (same variance reduction)
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    nf = 1 << 28
    wa = (0.5, 0.2, 0.8426149773176359)
    fur = {}
    for method, name in ((0, "cap"), (1, "heitz")):
        t = timed(lambda: vndf.vndf_furnace(method, wa, (0.3, 0.1), 17, nf, sums, stream=stream))
        torch.cuda.synchronize()
        s1, s2 = sums.cpu().tolist()
        fur[name] = (t, s1 / nf, s2 / nf - (s1 / nf) ** 2)
    nxt["furnace_t_heitz_over_t_cap"] = round(fur["heitz"][0] / fur["cap"][0], 4)
    nxt["furnace_estimate_var"] = [round(fur["cap"][1], 5), round(fur["cap"][2], 5),
                                   round(fur["heitz"][1], 5), round(fur["heitz"][2], 5)]
    # NEXT-3: device histogram throughput (2^28 samples into 64 x 64 bins)
    cnt = torch.zeros(64 * 64, dtype=torch.int64, device=dev)
    t_h = timed(lambda: vndf.vndf_histogram(0, 0, wa, (0.3, 0.1), 17, 1 << 28, 64, 64, cnt, stream=stream), 5)
    nxt["histogram_gsamples_s"] = gs(1 << 28, t_h)
    torch.cuda.empty_cache()
    res["next"] = nxt
    return res


def run_reference(args):
    """The tier's reference arm: the float64 oracle, as it stands, on this box's
    host cores; each step a bounded 2^22-sample slice (indices [0, 2^22)) of the
    config-4 workload.  Under torchrun only rank 0 runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    oracle.build()
    cfg = synth.CONFIGS[WORKLOAD_CID]
    m = 1 << 22
    idx = np.arange(m, dtype=np.uint64)
    threads = oracle.default_threads()
    for _ in range(args.warmup):
        oracle.batch_sample_philox(oracle.CAP, C4_SEED, idx, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.batch_sample_philox(oracle.CAP, C4_SEED, idx, threads=threads)
    dt = time.perf_counter() - t0
    value = m * args.steps / dt / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same recipe as ours)",
        "config": {"workload": f"config 4: {cfg.label}", "samples_per_step": m,
                   "note": "each step a bounded 2^22-sample slice of the 2^30-sample workload"},
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"config-4 indices [0, 2^22) per step, {threads} threads"},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
