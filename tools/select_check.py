"""Dev tool: the seed selection kernels against each other and the oracle on C0 (GPU)."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    import paper_2503_17911_b200 as vsag
    import synth
    c0 = synth.make_workload(synth.get_config("C0"), device="cuda", gt=False)
    dev = torch.device("cuda:0")
    xt = torch.from_numpy(c0["x"]).to(dev)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, torch.from_numpy(c0["entry"]).to(dev), adj=torch.from_numpy(c0["graph"]).to(dev))
    out = {}
    for ef in (1, 64, 128):
        ids, d, tr = ix.search(torch.from_numpy(c0["q"]).to(dev), 10, ef, 64 if ef < 64 else ef, trace=True,
                               max_hops=400, visited_slots=16384)
        for k, v in tr.items():
            out[f"{k}_{ef}"] = v.cpu().numpy()
    np.savez(sys.argv[2], **out)
    sys.exit(0)

import oracle  # noqa: E402
import synth  # noqa: E402
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "run", "/tmp/sel_new.npz"], check=True, env=env)
env["VSAG_SELECT_HIST"] = "1"
subprocess.run([sys.executable, __file__, "run", "/tmp/sel_old.npz"], check=True, env=env)
a, b = np.load("/tmp/sel_new.npz"), np.load("/tmp/sel_old.npz")
c0 = synth.make_workload(synth.get_config("C0"), device="cpu", gt=False)
lo, hi = oracle.train_sq(c0["x"])
codes = oracle.encode_sq(c0["x"], 8, lo, hi)
for ef in (1, 64, 128):
    o = oracle.search_batch(c0["x"], codes, lo, hi, 8, c0["graph"], c0["entry"], c0["q"], 10, ef, 64 if ef < 64 else ef,
                            trace=True, max_hops=400, nthreads=8)
    for key in ("hops", "n_lp", "pool_ids", "pool_tau", "expanded"):
        na, nb = a[f"{key}_{ef}"], b[f"{key}_{ef}"]
        bad_new = np.nonzero((na != o[key]).reshape(len(na), -1).any(1))[0]
        bad_old = np.nonzero((nb != o[key]).reshape(len(nb), -1).any(1))[0]
        print(f"ef={ef} {key}: new differs on {len(bad_new)} queries {bad_new[:8]}, old on {len(bad_old)} {bad_old[:8]}")
