"""BASELINE.json configs as seeded synthetic workloads.

No dataset is available offline; each config's graph is drawn by a seeded
generator with the shape BASELINE.json states, and X by a seeded stream
(UniformRng semantics, prng.hpp:11-28). Seeds follow SURVEY §8d:
graph 0xC0F60000+i, X 0xC0F61000+i, weights 0xC0F62000+i.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import (CbmMatrix, CsrBinaryMatrix, build_cbm, build_cbm_normalized, generate_dense,
               generate_graph)


@dataclass(frozen=True)
class Workload:
    name: str
    graph_kind: str
    graph_params: tuple
    normalized: bool
    d: int
    x_kind: str            # "int" (integers in [-8, 8]) or "normal" (N(0,1))
    alpha: int
    index: int
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def graph_seed(self):
        return 0xC0F60000 + self.index

    @property
    def x_seed(self):
        return 0xC0F61000 + self.index

    def graph(self) -> CsrBinaryMatrix:
        return generate_graph(self.graph_kind, list(self.graph_params), self.graph_seed)

    def build(self, a: CsrBinaryMatrix, threads: int) -> CbmMatrix:
        if self.normalized:
            return build_cbm_normalized(a, self.alpha, threads)
        return build_cbm(a, self.alpha, threads)

    def operand(self, n_rows: int, d: int | None = None, out=None):
        d = self.d if d is None else d
        if self.x_kind == "int":
            return generate_dense("int", n_rows, d, self.x_seed, -8, 8, out=out)
        return generate_dense("normal", n_rows, d, self.x_seed, out=out)


WORKLOADS = {
    "cfg0": Workload("cfg0", "community", (4096, 64, 0.5, 0.001), False, 64, "int", 0, 0,
                     "binary A.X, 64 communities of 64, p=0.5/0.001, X int [-8,8] (bit-exact gate)"),
    "cfg1": Workload("cfg1", "pa_triangle", (19717, 2, 0.3), True, 512, "normal", 0, 1,
                     "normalized A_hat.X, preferential attachment m=2 + 30% triangle closing"),
    "cfg2": Workload("cfg2", "clique_overlay", (235868, 1200000, 2, 10, 1.1), False, 128,
                     "normal", 8, 2,
                     "binary A.X, clique overlay 1.2M groups of 2..10, Zipf 1.1 popularity"),
    "cfg3": Workload("cfg3", "community", (132534, 500, 0.8, 1e-4), True, 256, "normal", 0, 3,
                     "normalized A_hat at d=256 (the GCN's A_hat products), communities of 500"),
    "cfg4_64": Workload("cfg4_64", "clique_overlay", (2449029, 4000000, 2, 16, 1.1), False, 64,
                        "normal", 8, 4, "scaling sweep, binary, d=64"),
}
