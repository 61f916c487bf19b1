"""Measurement beyond the bench line: ef sweeps of BASELINE.json configs C2, C3 and C4 (and C1)
at full size (C4 at a reduced N by default), recall@k against exact ground truth, the search
kernel's time and the whole step's, QPS, and the roofline of the search kernel on exact
counters.

python tools/config_sweep.py C2 C3 C4 [--c4n 2000000] > profiles/r02_config_sweep.json

Per (config, ef):
  - timed runs in the default configuration (visited cache chosen by the library);
  - one traced run with the exact visited set (visited_kind = "bitset": V never forgets), whose
    hops / n_lp / n_hp are Alg. 1's exact counters; B_q = 4d + hops*4R +
    (n_lp - |I|)*cb + n_hp*4d + 8k from them, and the re-evaluation rate of the default
    configuration (its n_lp over the exact one);
  - timed runs with the exact bitset as well (where it is the faster choice, e.g. C3);
  - the oracle (oracle/, the CPU transcription) on the host cores, 1 thread and all threads, on
    a bounded sample of the same queries.
Every config is built by synth (seeded, synthetic stand-ins).  C2 is also run
with NEXT-1 (99% truncated range + weighted L2).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17911_b200 as vsag  # noqa: E402
import synth  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


def b_q(cfg, tr, n_seed):
    d, R, k = cfg.d, cfg.degree, cfg.k
    cb = d if cfg.bits == 8 else (d + 1) // 2
    hops = tr["hops"].astype(np.float64)
    n_trav = tr["n_lp"].astype(np.float64) - n_seed
    nhp = tr["n_hp"].astype(np.float64)
    return 4 * d + hops * 4 * R + n_trav * cb + nhp * 4 * d + 8 * k


def oracle_qps(w, cfg, metric, ef, rr, lo, hi, codes, nthreads, budget):
    import oracle
    x, q = w["x"], w["q"]
    args = (x, codes, lo, hi, cfg.bits, w["graph"], w["entry"])
    m = min(len(q), max(4, nthreads))
    t = time.perf_counter()
    oracle.search_batch(*args, q[:m], cfg.k, ef, rr, metric, nthreads=nthreads)
    per = (time.perf_counter() - t) / m
    m2 = int(min(len(q), max(m, budget / max(per, 1e-9))))
    t = time.perf_counter()
    oracle.search_batch(*args, q[:m2], cfg.k, ef, rr, metric, nthreads=nthreads)
    dt = time.perf_counter() - t
    return {"qps": round(m2 / dt, 1), "threads": nthreads, "sample_queries": m2, "seconds": round(dt, 2)}


def sweep(cfg, w, variants, reps=5, oracle_budget=3.0, with_oracle=True):
    dev = torch.device("cuda:0")
    torch.cuda.empty_cache()  # (the graph build's cached blocks would starve the library's own pool)
    xt = torch.from_numpy(w["x"]).to(dev)
    qd = torch.from_numpy(w["q"]).to(dev)
    nq = len(w["q"])
    n_seed = len(np.unique(w["entry"]))
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    peak = peak_gbs()
    out = {}
    for name, (metric, quantile) in variants.items():
        lo, hi = vsag.train_sq(xt, quantile)
        codes, _, _ = vsag.encode_sq(xt, cfg.bits, lo, hi)
        ix = vsag.Index(xt, codes, lo, hi, cfg.bits, torch.from_numpy(w["entry"]).to(dev),
                        adj=torch.from_numpy(w["graph"]).to(dev))
        import oracle
        lo_n, hi_n = lo.cpu().numpy(), hi.cpu().numpy()
        ocodes = oracle.encode_sq(w["x"], cfg.bits, lo_n, hi_n)
        res = {}
        for ef in cfg.efs:
            rr = cfg.rerank_n(ef)
            r = {}
            for kind in ("auto", "bitset"):
                torch.cuda.empty_cache()
                ix.search(qd, cfg.k, ef, rr, metric, visited_kind=kind)
                tt, ts = [], []
                for _ in range(reps):
                    flush.zero_()
                    ids, _, tm = ix.search(qd, cfg.k, ef, rr, metric, timing=True, visited_kind=kind)
                    tt.append(tm["ms_total"])
                    ts.append(tm["ms_search"])
                _, _, tr = ix.search(qd, cfg.k, ef, rr, metric, trace=True, visited_kind=kind)
                tr = {k2: v.cpu().numpy() for k2, v in tr.items()}
                r[kind] = dict(step_ms=round(float(np.median(tt)), 4), search_ms=round(float(np.median(ts)), 4),
                               qps=round(nq / float(np.median(tt)) * 1e3), n_lp=round(float(tr["n_lp"].mean()), 1),
                               n_miss=round(float(tr["n_miss"].mean()), 2), visited_kind=tm["visited_kind"],
                               visited_slots=tm["visited_slots"])
                if kind == "bitset":
                    assert int(tr["n_miss"].sum()) == 0
                    bq = b_q(cfg, tr, n_seed)
                    r["exact"] = dict(hops=round(float(tr["hops"].mean()), 1), n_lp=round(float(tr["n_lp"].mean()), 1),
                                      n_hp=round(float(tr["n_hp"].mean()), 1), B_q=round(float(bq.mean())))
                    rec = synth.recall_at_k(ids.cpu().numpy(), w["gt"], cfg.k)
            ex = r["exact"]
            r["recall"] = round(rec, 4)
            r["reevaluation_rate_auto"] = round(r["auto"]["n_lp"] / ex["n_lp"] - 1.0, 4)
            best = min(("auto", "bitset"), key=lambda k2: r[k2]["step_ms"])
            bytes_launch = ex["B_q"] * nq
            r["roofline"] = {"kernel": "search_kernel", "config": best,
                             "GBs": round(bytes_launch / (r[best]["search_ms"] / 1e3) / 1e9, 1),
                             "frac": round(bytes_launch / (r[best]["search_ms"] / 1e3) / 1e9 / peak, 4),
                             "peak_GBs": peak}
            none = {"qps": None}
            r["oracle_1t"] = oracle_qps(w, cfg, metric, ef, rr, lo_n, hi_n, ocodes, 1, oracle_budget) if with_oracle else none
            r["oracle_pt"] = (oracle_qps(w, cfg, metric, ef, rr, lo_n, hi_n, ocodes, os.cpu_count() or 1, oracle_budget)
                              if with_oracle else none)
            res[ef] = r
            log(f"  {cfg.name} {name} ef={ef} recall={r['recall']} auto={r['auto']} bitset={r['bitset']} "
                f"exact={ex} roofline={r['roofline']} oracle1={r['oracle_1t']['qps']} oracleP={r['oracle_pt']['qps']}")
        out[name] = res
        ix.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--c4n", type=int, default=2_000_000)
    ap.add_argument("--no-oracle", action="store_true", help="skip the oracle timings (A/B runs)")
    args = ap.parse_args()
    report = {"gpu": torch.cuda.get_device_name(0), "host_threads": os.cpu_count()}
    for name in args.configs:
        cfg = synth.get_config(name)
        if name == "C4" and args.c4n != cfg.n:
            cfg = cfg.scaled(n=args.c4n)
        t = time.time()
        w = synth.make_workload(cfg, device="cuda", gt=True, log=log)
        log(f"[{cfg.name}] workload {time.time() - t:.0f} s")
        if name == "C2":
            variants = {"sq4_l2": ("l2", 1.0), "sq4_l2w_q99": ("l2w", 0.99)}
        else:
            variants = {f"sq{cfg.bits}_{cfg.metric}": (cfg.metric, 1.0)}
        report[cfg.name] = dict(n=cfg.n, d=cfg.d, nq=cfg.nq, k=cfg.k, degree=cfg.degree, bits=cfg.bits,
                                seeds=cfg.n_seeds, results=sweep(cfg, w, variants, with_oracle=not args.no_oracle))
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
