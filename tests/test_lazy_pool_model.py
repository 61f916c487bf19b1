"""Host-side model of the search kernel's lazy pool against Alg. 1 as written.

The kernel does not insert a hop's new keys into the sorted pool at once: they stay in an unsorted
pending buffer and are merged in batches, and the next expansion is chosen from the pool's first
unexpanded entry (rank sel + pexp) and the smallest unexpanded pending key (rank = pool lower bound
+ expanded pending keys below it).  This test runs that selection rule, written out in plain Python
exactly as DESIGN.md §6.1 states it, next to the direct transcription of Alg. 1 (PAPER.md:348-389:
insert every key immediately, keep |C| <= L, expand the first unexpanded entry of the window) on
random graphs with random integer distances, and requires the same expansion sequence, hop count
and final pool for many (ef, L, buffer size, seed count) combinations, including buffers so small
that every hop merges and windows much smaller than the pool.  It shares no code with the CUDA path
or the oracle; it pins the argument, not the implementation.
"""
import bisect
import random

import pytest


def make_case(rng, n, degree):
    graph = [rng.sample(range(n), degree) for _ in range(n)]
    tau = [rng.randrange(0, 4 * n) for _ in range(n)]  # ties happen: keys are (tau, id)
    return graph, tau


def alg1_reference(graph, tau, seeds, ef, L):
    """Alg. 1 with the readings R-8/R-9/R-10/R-14: sorted pool of (tau, id), capacity L, window ef."""
    pool = sorted((tau[s], s) for s in seeds)[:L]
    expanded = set()
    visited = {i for _, i in pool}
    order = []
    while True:
        sel = next((k for k in pool[:ef] if k[1] not in expanded), None)
        if sel is None:
            break
        expanded.add(sel[1])
        order.append(sel[1])
        for j in graph[sel[1]]:
            if j in visited:
                continue
            visited.add(j)
            bisect.insort(pool, (tau[j], j))
            del pool[L:]
    return order, pool


def lazy_pool(graph, tau, seeds, ef, L, cap):
    """The kernel's rule: pool P stays as it was after the last merge, new keys go to `pend`."""
    P = sorted((tau[s], s) for s in seeds)[:L]
    flag = {}            # key -> expanded (for keys in P and in pend)
    pend = []            # unsorted pending keys
    pexp = 0             # expanded pending keys
    visited = {i for _, i in P}
    order = []

    def merge():
        nonlocal P, pend, pexp
        P = sorted(P + pend)[:L]
        pend, pexp = [], 0

    while True:
        lim = min(ef - pexp, len(P))
        sel = next((t for t in range(max(lim, 0)) if not flag.get(P[t], False)), None)
        ks = P[sel] if sel is not None else None
        unexp = [k for k in pend if not flag.get(k, False)]
        pmink = min(unexp) if unexp else None
        if pmink is not None and (ks is None or pmink < ks):
            cnt = sum(1 for k in pend if flag.get(k, False) and k < pmink)
            wpos = ef - cnt - 1
            if wpos < 0 or (wpos < len(P) and not pmink < P[wpos]):
                break
            key = pmink
            pexp += 1
        else:
            if ks is None:
                break
            key = ks
        flag[key] = True
        order.append(key[1])
        new = []
        for j in graph[key[1]]:
            if j not in visited:
                visited.add(j)
                new.append(j)
        if pend and len(pend) + len(new) > cap:
            merge()
        worst = P[L - 1] if len(P) == L else None  # stale between merges: never too tight
        for j in new:
            k = (tau[j], j)
            if worst is None or k < worst:
                pend.append(k)
        assert len(pend) <= max(cap, len(new))
    merge()
    return order, P


@pytest.mark.parametrize("ef,L,cap,nseed", [(1, 1, 8, 3), (1, 10, 8, 5), (2, 50, 8, 40), (8, 8, 8, 8), (8, 64, 16, 4),
                                            (16, 16, 8, 32), (33, 97, 32, 16), (64, 64, 32, 64), (40, 300, 32, 7),
                                            (5, 5, 1, 2)])
def test_lazy_pool_rule_equals_alg1(ef, L, cap, nseed):
    for seed in range(25):
        rng = random.Random(1000 * ef + seed)
        n, degree = 400, 8
        graph, tau = make_case(rng, n, degree)
        seeds = rng.sample(range(n), nseed)
        ro, rp = alg1_reference(graph, tau, seeds, ef, L)
        lo, lp = lazy_pool(graph, tau, seeds, ef, L, max(cap, degree))
        assert lo == ro, f"expansion order differs (seed {seed})"
        assert lp == rp, f"final pool differs (seed {seed})"
        assert len(ro) > 0
