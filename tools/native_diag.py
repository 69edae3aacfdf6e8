import sys, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import oracle, synth, paper_2306_05044_b200 as vndf
dev = torch.device("cuda:0")
n = 1 << 22
x = synth.fill(5, 4, n, device=dev)
out = vndf.empty_outputs(n, dev)
vndf.vndf_sample_cap_pdf_native(*[x[k] for k in synth.PLANES], *out)
torch.cuda.synchronize()
host = [x[k].cpu().numpy() for k in synth.PLANES]
h_ref, p_ref = oracle.batch_sample_native(oracle.CAP, *host)
h = np.stack([o.cpu().numpy() for o in out[:3]]).astype(np.float64)
eh = np.abs(h - h_ref).max(axis=0)
ep = np.abs(out[3].cpu().numpy() - p_ref) / p_ref
print("max", eh.max(), ep.max(), (eh > 2e-5).sum(), (ep > 1e-4).sum())
for k in np.argsort(-eh)[:5]:
    wi = np.array([host[0][k], host[1][k], host[2][k]], dtype=np.float64)
    ax, ay = float(host[3][k]), float(host[4][k])
    t = np.array([ax * wi[0], ay * wi[1], wi[2]]); ws = t / np.linalg.norm(t)
    print(json.dumps({"dh": float(eh[k]), "dp": float(ep[k]), "in": [float(v[k]) for v in host], "wsz": float(ws[2]), "h": h[:, k].tolist(), "ref": h_ref[:, k].tolist()}))
for k in np.argsort(-ep)[:3]:
    print("pdf", float(ep[k]), [float(v[k]) for v in host])
