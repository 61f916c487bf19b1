"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no SQ training/encoding, no
tau_l, no greedy search, no rerank).  It only produces the *inputs* of the hot
path -- base vectors, queries, the fixed-degree proximity graph (construction is
out of scope, BASELINE.json north_star: "Graph construction ... out of scope
except as input preparation") and the entry set -- plus the exact brute-force
ground truth used to measure recall (Recall@k definition).

Workload recipes follow SURVEY.md §8(d).1 (stand-ins for the paper's datasets,
PAPER.md:654-681 Table 3; none of their records are reproduced):

  C0  10k x 128, 10-component Gaussian mixture (means U[-1,1], sigma 0.3)
  C1  1M x 128, integer Gamma-mixture in [0,255] (SIFT1M-shaped)
  C2  1M x 960, 1000-cluster mixture, per-dim scales U[0.05,1] (GIST1M-shaped)
  C3  1M x 768 unit vectors, 512-cluster vMF-like mixture (embedding-shaped)
  C4  10M x 96 unit vectors, 4096-cluster mixture (large batch)

All generation uses numpy.random.Generator(PCG64(seed)) in float64 and casts to
float32 at the end.  Base rows: seed 0; queries: seed 1 (cluster parameters are
re-drawn from seed 0 so queries follow the same mixture); entry sets: seed 2.
Rows are drawn in 1M-row chunks in row order so the stream order is defined.
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .generators import generate_base, generate_queries, entry_set  # noqa: F401
from .graph import build_graph, build_labelled_graph, knn_candidates, rng_prune_fill  # noqa: F401
from .groundtruth import ground_truth, recall_at_k  # noqa: F401
from .workload import make_workload  # noqa: F401
