import json, sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import oracle, synth, paper_2306_05044_b200 as vndf
dev = torch.device("cuda:0")
for cid in (2, 5):
    cfg = synth.CONFIGS[cid]; n = 1 << 22
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    out = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_heitz2018(*[x[k] for k in synth.PLANES], *out)
    torch.cuda.synchronize()
    host = [x[k].cpu().numpy() for k in synth.PLANES]
    h_ref, p_ref, ti = oracle.batch_sample(oracle.HEITZ, *host)
    h = np.stack([o.cpu().numpy() for o in out[:3]]).astype(np.float64)
    eh = np.abs(h - h_ref).max(axis=0)
    ax, ay = host[3].astype(np.float64), host[4].astype(np.float64)
    s = np.where(host[2] < 0, -1.0, 1.0)
    N = 1 / np.sqrt((s * h_ref[0] / ax) ** 2 + (s * h_ref[1] / ay) ** 2 + h_ref[2] ** 2)
    rim = 1.0 - host[6].astype(np.float64) * np.cos(2 * np.pi * host[5].astype(np.float64)) ** 2
    good = (ti >= 0.05) & (N >= 0.1 * np.maximum(ax, ay)) & (rim >= 2.5e-3)
    for k in np.argsort(-np.where(good, eh, 0))[:6]:
        print(json.dumps({"cid": cid, "dh": float(eh[k]), "ti": float(ti[k]), "N/amax": float(N[k] / max(ax[k], ay[k])), "rim": float(rim[k]),
              "in": [float(v[k]) for v in host], "h": h[:, k].tolist(), "ref": h_ref[:, k].tolist()}))
