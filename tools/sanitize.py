"""Drive every libvsag kernel variant on small inputs, for compute-sanitizer runs.

    VSAG_CACHE_DIR=/tmp/vsag_cache python tools/sanitize.py --prep      # build inputs (no sanitizer)
    compute-sanitizer --tool memcheck --kernel-name regex:vsag python tools/sanitize.py [--c1 1000]
    VSAG_LIB_VARIANT=chk python tools/sanitize.py      # the bounds-checked build (VSAG_CHECKS)

Covers: SQ train / encode / truncated train, index load (fixed-degree, CSR, layout 1, PRS
delta, labels), query prep, the tcgen05 seed contraction (L2 / IP, SQ8 / SQ4), the dp4a seed
tile (weighted L2), seed selection, and the search kernel in its compile-time common case
(with and without trace) and the generic variant: u16 / u32 / bitset visited sets, degree 64
(two id slices, the de-duplicating merge), CSR, layout 1, PRS blocks, label filter, QLP,
adaptive re-rank, code-lane shapes, SQ4, IP and weighted L2.  C0 (10k x 128) and a slice of
C1's queries (1M x 128).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prep", action="store_true", help="only build and cache the inputs")
    ap.add_argument("--c1", type=int, default=1000, help="C1 queries searched (0: skip C1)")
    args = ap.parse_args()
    c0 = synth.make_workload(synth.get_config("C0"), device="cuda", csr=True, gt=False)
    c3s = synth.make_workload(synth.get_config("C3").scaled(n=8000, nq=48, clusters=64), device="cuda", gt=False)
    c1 = synth.make_workload(synth.get_config("C1"), device="cuda", gt=False) if args.c1 else None
    lab_cfg = synth.get_config("C0").scaled(n=1500, nq=40, clusters=3, n_seeds=48)
    lw = synth.make_workload(lab_cfg, device="cpu", gt=False)
    if args.prep:
        print("inputs cached")
        return
    import paper_2503_17911_b200 as vsag
    dev = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    runs = 0

    def searches(ix, q, k, ef, rr, metric="l2", **extra):
        # timing=True synchronises and reads the index's device flag: with the bounds-checked
        # build (VSAG_LIB_VARIANT=chk) a failed check raises VsagError here
        nonlocal runs
        ix.search(q, k, ef, rr, metric, timing=True, **extra)
        ix.search(q, k, ef, rr, metric, trace=True, max_hops=ef + 64, timing=True, **extra)
        runs += 2

    # ---- C0: every search-kernel variant
    xt, q = t(c0["x"]), t(c0["q"])
    for bits in (8, 4):
        codes, lo, hi = vsag.encode_sq(xt, bits)
        for layout in ("table", "colocated"):
            ix = vsag.Index(xt, codes, lo, hi, bits, t(c0["entry"]), adj=t(c0["graph"]), layout=layout)
            for metric in ("l2", "ip", "l2w"):
                searches(ix, q, 10, 64, 64, metric)
            searches(ix, q, 10, 64, 64, visited_slots=256)
            searches(ix, q, 10, 64, 64, visited_kind="u32")
            searches(ix, q, 10, 64, 64, visited_kind="bitset")
            searches(ix, q, 10, 64, 64, code_lanes=8)
            searches(ix, q, 10, 200, 200)
            searches(ix, q[:7], 3, 1, 10)
            ix.close()
        ixc = vsag.Index(xt, codes, lo, hi, bits, t(c0["entry"]), adj=t(c0["col"]), row_ptr=t(c0["row_ptr"]),
                         degree=32)
        searches(ixc, q, 10, 64, 64)
        ixc.set_prs(0.5)
        searches(ixc, q, 10, 64, 64)
        searches(ixc, q, 10, 64, 64, qlp=(8, 24, 1, 10 ** 6))
        ixc.close()
    codes, lo, hi = vsag.encode_sq(xt, 8)
    ix = vsag.Index(xt, codes, lo, hi, 8, t(c0["entry"]), adj=t(c0["graph"]))
    searches(ix, q, 10, 64, 64, rerank_adaptive=False, qlp=(3, 12, 2, 10 ** 5))
    ix.close()
    lo2, hi2 = vsag.train_sq(xt, 0.99)
    codes2, _, _ = vsag.encode_sq(xt, 8, lo2, hi2)
    ix = vsag.Index(xt, codes2, lo2, hi2, 8, t(c0["entry"]), adj=t(c0["graph"]))
    searches(ix, q, 10, 64, 64, "l2w")
    ix.close()
    # adaptive re-rank needs every base value inside the range (C1-like integer data)
    cfg_a = synth.get_config("C1").scaled(n=4000, nq=40, clusters=4, n_seeds=64)
    wa = synth.make_workload(cfg_a, device="cuda", gt=False)
    xa = wa["x"].copy()
    xa[0], xa[1] = 0.0, 255.0
    xat = t(xa)
    codes, lo, hi = vsag.encode_sq(xat, 8)
    ix = vsag.Index(xat, codes, lo, hi, 8, t(wa["entry"]), adj=t(wa["graph"]))
    searches(ix, t(wa["q"]), 10, 64, 64, rerank_adaptive=True)
    ix.close()
    # label filter (NEXT-2)
    adj, lab = synth.build_labelled_graph(lw["x"], 24)
    xl = t(lw["x"])
    codes, lo, hi = vsag.encode_sq(xl, 8)
    ix = vsag.Index(xl, codes, lo, hi, 8, t(lw["entry"]), adj=t(adj))
    ix.set_labels(t(lab))
    searches(ix, t(lw["q"]), 10, 40, 40, max_degree=12, alpha_s=1.2)
    ix.close()
    # degree 64: E = 2, forgetful caches (de-duplicating merge), both layouts, SQ8 / SQ4
    x3 = t(c3s["x"])
    for bits in (8, 4):
        codes, lo, hi = vsag.encode_sq(x3, bits)
        for layout in ("table", "colocated"):
            ix = vsag.Index(x3, codes, lo, hi, bits, t(c3s["entry"]), adj=t(c3s["graph"]), layout=layout)
            for kind, slots in (("u16", 256), ("u32", 256), ("bitset", 0), ("auto", 0)):
                searches(ix, t(c3s["q"]), 100, 128, 128, "ip", visited_kind=kind, visited_slots=slots)
            searches(ix, t(c3s["q"]), 10, 64, 64, "l2")
            ix.close()
    # ---- C1 slice: the bench's configuration (common-case variant) and the u32 table
    if c1 is not None:
        x1 = t(c1["x"])
        codes, lo, hi = vsag.encode_sq(x1, 8)
        ix = vsag.Index(x1, codes, lo, hi, 8, t(c1["entry"]), adj=t(c1["graph"]))
        q1 = t(c1["q"][: args.c1])
        searches(ix, q1, 10, 132, 132)
        searches(ix, q1, 10, 132, 132, visited_slots=256)
        searches(ix, q1, 10, 132, 132, visited_kind="bitset")
        hq = torch.from_numpy(c1["q"][: args.c1]).pin_memory()
        ix.search_host(hq, 10, 132, 132)
        ix.close()
    torch.cuda.synchronize()
    print(f"sanitize driver done: {runs} searches")


if __name__ == "__main__":
    main()
