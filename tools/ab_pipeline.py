"""Dev tool: A/B of library builds on C1 at one ef, in one process per variant.

    VSAG_LIB_VARIANT=base python tools/ab_pipeline.py --ef 130     # libvsag_base.so
    python tools/ab_pipeline.py --ef 130                            # libvsag.so

Prints the per-stage standalone times (L2 flushed before each call; medians) and the
pipelined step time of bench.py's timed loop (2 streams, 4 rotating 10k-query sets).
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ef", type=int, default=130)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--layout", default="table", choices=["table", "colocated"])
    ap.add_argument("--prs", type=float, default=0.0, help="PRS delta on a table index (0: none)")
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--wpb", type=int, default=int(os.environ.get("VSAG_AB_WPB", "0")), help="warps per block (0: default)")
    args = ap.parse_args()
    cfg = synth.get_config("C1")
    w = synth.make_workload(cfg, device="cuda", gt=False)
    dev = torch.device("cuda:0")
    xt = torch.from_numpy(w["x"]).to(dev)
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, torch.from_numpy(w["entry"]).to(dev), adj=torch.from_numpy(w["graph"]).to(dev),
                    layout=args.layout)
    if args.prs > 0:
        ix.set_prs(args.prs)
    nq = len(w["q"])
    qsets = [torch.from_numpy(w["q"]).to(dev)] + [
        torch.from_numpy(synth.generate_queries(cfg, nq, seed=100 + i)).to(dev) for i in range(1, 4)]
    ef = args.ef
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    name = os.environ.get("VSAG_LIB_VARIANT", "new") + f" {args.layout}" + (f" prs={args.prs}" if args.prs else "") + \
        f" streams={args.streams} wpb={args.wpb}"
    for _ in range(3):
        ix.search(qsets[0], 10, ef, ef, warps_per_block=args.wpb)
    st = {"prep": [], "seed": [], "search": [], "total": []}
    for i in range(args.reps):
        flush.zero_()
        _, _, tm = ix.search(qsets[i % 4], 10, ef, ef, timing=True, warps_per_block=args.wpb)
        st["prep"].append(tm["ms_query_prep"])
        st["seed"].append(tm["ms_seed"])
        st["search"].append(tm["ms_search"])
        st["total"].append(tm["ms_total"])
    med = {k: statistics.median(v) for k, v in st.items()}
    ns = args.streams
    streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    outs = [(torch.empty((nq, 10), dtype=torch.int32, device=dev), torch.empty((nq, 10), device=dev)) for _ in range(ns)]
    main_s = torch.cuda.current_stream(dev)
    res = []
    for _ in range(args.rounds):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        for s in streams:
            s.wait_event(a)
        for i in range(args.steps):
            with torch.cuda.stream(streams[i % ns]):
                ix.search(qsets[i % 4], 10, ef, ef, out=outs[i % ns], warps_per_block=args.wpb)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)
        b.record(main_s)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / args.steps)
    pm = min(res)
    print(f"[{name}] ef={ef} standalone: prep {med['prep']:.4f} seed {med['seed']:.4f} search {med['search']:.4f} "
          f"total {med['total']:.4f} ms | pipelined step {pm:.4f} ms ({nq / pm * 1e3 / 1e6:.2f} M QPS) "
          f"rounds {[round(r, 4) for r in res]}", flush=True)
    ix.close()


if __name__ == "__main__":
    main()
