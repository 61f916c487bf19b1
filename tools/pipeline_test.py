"""Dev tool: back-to-back C1 steps on one stream vs alternating two streams (batch pipelining)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config("C1")
w = synth.make_workload(cfg, device="cuda", gt=False)
dev = torch.device("cuda:0")
xt = torch.from_numpy(w["x"]).to(dev)
codes, lo, hi = vsag.encode_sq(xt, 8)
ix = vsag.Index(xt, codes, lo, hi, 8, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev))
q = torch.from_numpy(w["q"]).to(dev)
nq = q.shape[0]
K = 40
for ns in (1, 2, 3):
    streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    outs = [(torch.empty((nq, 10), dtype=torch.int32, device=dev), torch.empty((nq, 10), device=dev)) for _ in range(ns)]
    for it in range(2):
        main = torch.cuda.current_stream(dev)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(main)
        for s in streams:
            s.wait_event(start)
        for i in range(K):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                ix.search(q, 10, 160, 160, out=outs[i % ns])
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        end.record(main)
        torch.cuda.synchronize()
        ms = start.elapsed_time(end) / K
    print(f"streams={ns}: {ms:.3f} ms/step  {nq / ms * 1e3 / 1e6:.2f} M QPS", flush=True)
