"""BASELINE.json configs C0-C4 as data (SURVEY.md §8(a) shape table, §8(d).1).

`rerank` is the rule for R' (the number of pool entries re-ranked in fp32,
Alg. 1 line 18): "ef" means R' = ef (AMB-15), "2ef" means
R' = 2*ef (BASELINE.json config 2), an int is a fixed count (config 0: 64).
"""
from __future__ import annotations

import dataclasses
from typing import Tuple, Union


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    kind: str            # generator family: gauss10 | gamma_int | scaled_mix | sphere
    n: int               # base vectors
    d: int               # dimension
    nq: int              # queries
    degree: int          # graph out-degree R
    bits: int            # SQ bits (8 or 4)
    metric: str          # "l2" | "ip"
    k: int
    efs: Tuple[int, ...]
    rerank: Union[str, int]
    n_seeds: int         # |I| (AMB-11)
    clusters: int
    sigma: float

    def rerank_n(self, ef: int) -> int:
        if self.rerank == "ef":
            return ef
        if self.rerank == "2ef":
            return 2 * ef
        return int(self.rerank)

    def scaled(self, n: int | None = None, nq: int | None = None,
               clusters: int | None = None, n_seeds: int | None = None) -> "Config":
        """A smaller instance with the same generator and structure (for tests)."""
        return dataclasses.replace(
            self,
            name=f"{self.name}-n{n or self.n}-q{nq or self.nq}",
            n=n or self.n, nq=nq or self.nq,
            clusters=clusters or self.clusters,
            n_seeds=min(n_seeds or self.n_seeds, n or self.n))


CONFIGS = {
    # config 0 (BASELINE.json): 10-component Gaussian mixture, sigma 0.3; SQ8; k=10, ef=64, top-64 rerank.
    "C0": Config("C0", "gauss10", 10_000, 128, 100, 32, 8, "l2", 10, (64,), 64, 128, 10, 0.3),
    # config 1: 1M x 128 integer Gamma(0.5,30) 100-cluster mixture; SQ8 + fp32 rerank; ef sweep.
    # 130..192 added: finer steps around the recall@10 >= 0.95 crossing.
    "C1": Config("C1", "gamma_int", 1_000_000, 128, 10_000, 32, 8, "l2", 10,
                 (16, 32, 64, 128, 130, 132, 134, 136, 144, 152, 160, 192, 256), "ef", 1024, 100, 0.0),
    # config 2: 1M x 960, 1000 clusters, per-dim scales U[0.05,1]; SQ4; rerank top 2*ef.
    "C2": Config("C2", "scaled_mix", 1_000_000, 960, 1_000, 32, 4, "l2", 10, (64, 128, 256), "2ef",
                 16384, 1000, 0.5),
    # config 3: 1M x 768 unit vectors, 512 clusters, sigma 0.2 per coordinate; SQ8 IP; k=100.
    "C3": Config("C3", "sphere", 1_000_000, 768, 10_000, 64, 8, "ip", 100, (128, 256, 512), "ef",
                 256, 512, 0.2),
    # config 4: 10M x 96 unit vectors, 4096 clusters (sigma 0.2, SURVEY AMB-24); SQ4 L2; 100k queries.
    "C4": Config("C4", "sphere", 10_000_000, 96, 100_000, 32, 4, "l2", 10, (32, 64, 128), "ef",
                 256, 4096, 0.2),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]
