"""Write profiles/<round>/prof_c4_<round>_summary.txt and the fused kernels'
instruction counts and pipe utilisation in profiles/traffic.json from an
`ncu --set full` capture of `tools/prof_kernels.py c4` (2^26 samples per launch).

python tools/c4_profile_summary.py r1 gpurun_out/prof_c4_r1.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

rnd, rep = sys.argv[1], sys.argv[2]
N = 1 << 26
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
data = rows[2:]
EXTRA = ["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
PIPES = {"issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "fma_inst": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
         "fmaheavy_cycles": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "alu": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
         "xu_sfu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"}
res = ncu_summary.load(rep)
tpath = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(tpath))
out = os.path.join(ROOT, "profiles", rnd, f"prof_c4_{rnd}_summary.txt")
with open(out, "w") as f:
    f.write(f"ncu --set full summary of {os.path.basename(rep)} (tools/prof_kernels.py c4: 2^26 samples per launch)\n")
    for j, d in enumerate(res):
        f.write(d["kernel"] + "\n")
        for k, v in d.items():
            if k != "kernel":
                f.write(f"    {k:85s} {v}\n")
        for k in EXTRA:
            f.write(f"    {k:85s} {data[j][hdr.index(k)]}\n")
        ipw = float(str(d["smsp__inst_executed.sum"]).split()[0]) / N
        f.write(f"    {'warp-instructions per sample':85s} {ipw:.4f}\n")
        name = "cap" if "philox_kernel<0" in d["kernel"] else "heitz"
        traffic[f"{name}_philox_c4_warp_inst_per_sample"] = round(ipw, 4)
        traffic[f"{name}_philox_c4_pipes"] = {k: round(float(data[j][hdr.index(v)]) / 100, 4) for k, v in PIPES.items()}

# dynamic opcode counts per sample from the source page -> the FMA-datapath bound
# (DESIGN.md s.6.5): IMAD.WIDE 4.335 clk, FP32 FMA-pipe instruction 1.03 clk, other
# IMAD 2 clk per warp-instruction (tools/mix_probe.cu, tools/pipe_probe.cu)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True).stdout.decode("latin-1")
rows = list(csv.reader(io.StringIO(src)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
FP32 = ("FFMA", "FMUL", "FADD", "HFMA2", "FMUL.RZ", "FFMA.RZ", "FADD.FTZ", "FMUL.FTZ", "FFMA.FTZ")
rates = traffic.get("fma_pipe_rates_measured", {})
rates.setdefault("imad_wide_clk", 4.335)
rates.setdefault("ffma_clk", 1.03)          # FMUL, FADD, FFMA with an immediate or constant operand
rates.setdefault("ffma_3reg_clk", 1.52)     # FFMA with three register sources (tools/pipe_probe.cu: 0.656/clk)
rates.setdefault("imad_clk", 2.0)
traffic["fma_pipe_rates_measured"] = rates


def _three_regs(src: str) -> bool:
    """FFMA Rd, Ra, Rb, Rc (no immediate, constant-bank or RZ source)."""
    ops = src.split(None, 1)[1] if " " in src else ""
    args = [a.strip().lstrip("-|").rstrip("|") for a in ops.rstrip(";").split(",")]
    return len(args) == 4 and all(a.startswith("R") and a != "RZ" for a in args[1:])
done = set()
with open(out, "a") as f:
    for k, st in enumerate(starts):
        if rows[st][1] in done:     # the source page may list a kernel more than once
            continue
        done.add(rows[st][1])
        end = starts[k + 1] if k + 1 < len(starts) else len(rows)
        blk = rows[st + 1:end]
        col = {h: i for i, h in enumerate(blk[0])}
        ic = [h for h in blk[0] if "Instructions Executed" in h][0]
        wide = fp = fp3 = imad = 0.0
        for r in blk[1:]:
            if len(r) < len(blk[0]):
                continue
            t = r[col["Source"]].split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") else t[0]
            try:
                c = float(r[col[ic]] or 0)
            except ValueError:
                continue
            if op.startswith("IMAD.WIDE"):
                wide += c
            elif op.startswith("IMAD"):
                imad += c
            elif op.split(".")[0] == "FFMA" and _three_regs(" ".join(t[1:] if t[0].startswith("@") else t)):
                fp3 += c
            elif op in FP32 or op.split(".")[0] in ("FFMA", "FMUL", "FADD", "HFMA2"):
                fp += c
        ws = N / 32.0
        mix = {"IMAD.WIDE.U32": round(wide / ws, 2), "fp32_fma_pipe": round(fp / ws, 2),
               "ffma_3reg": round(fp3 / ws, 2), "IMAD_other": round(imad / ws, 2)}
        cyc = mix["IMAD.WIDE.U32"] * rates["imad_wide_clk"] + mix["fp32_fma_pipe"] * rates["ffma_clk"] + \
            mix["ffma_3reg"] * rates["ffma_3reg_clk"] + mix["IMAD_other"] * rates["imad_clk"]
        name = "cap" if "(int)0" in rows[st][1] or "philox_kernel<0" in rows[st][1] else "heitz"
        traffic[f"{name}_philox_c4_fma_mix"] = mix
        traffic[f"{name}_philox_c4_fma_pipe_cycles_per_warp_sample"] = round(cyc, 1)
        f.write(f"{name}: per 32 samples {mix} -> FMA datapath {cyc:.1f} clk\n")
json.dump(traffic, open(tpath, "w"), indent=1)
print(open(out).read())
