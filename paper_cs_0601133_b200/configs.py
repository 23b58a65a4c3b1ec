"""BASELINE.json's five fgemm workloads (names c1..c5 follow SURVEY.md §8(a)).

Pure data: shapes, primes, scalars and the generator seed of each config.
Inputs are drawn with the ffgen recipe (seed = config number, streams A=0,
B=1, C=2); C is generated only when beta != 0 (otherwise it is write-only).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    p: int
    m: int
    n: int
    k: int
    transA: str
    transB: str
    alpha: int
    beta: int
    seed: int
    gpus: tuple
    text: str

    @property
    def a_shape(self):
        return (self.m, self.k) if self.transA == "N" else (self.k, self.m)

    @property
    def b_shape(self):
        return (self.k, self.n) if self.transB == "N" else (self.n, self.k)

    def useful_ops(self) -> float:
        return 2.0 * self.m * self.n * self.k


CONFIGS = {
    "c1": Config("c1", 65521, 512, 512, 512, "N", "N", 1, 0, 1, (1,),
                 "ff_gemm p=65521, m=n=k=512, alpha=1, beta=0, NN, 1 GPU"),
    "c2": Config("c2", 8388593, 4096, 4096, 4096, "N", "N", 3, 1, 2, (1,),
                 "ff_gemm p=8388593 (largest prime < 2^23), m=n=k=4096, alpha=3, beta=1, NN, 1 GPU"),
    "c3": Config("c3", 251, 8192, 8192, 16384, "T", "N", 1, 0, 3, (1, 8),
                 "ff_gemm p=251, m=n=8192, k=16384, alpha=1, beta=0, transA=T, 1 and 8 GPUs"),
    "c4": Config("c4", 65521, 32768, 32768, 8192, "N", "N", 1, 0, 4, (1, 2, 4, 8),
                 "ff_gemm p=65521, m=n=32768, k=8192, alpha=1, beta=0, NN, row-panel sharded 1/2/4/8 GPUs"),
    "c5": Config("c5", 67108859, 16384, 16384, 16384, "N", "N", 67108858, 1, 5, (1, 2, 4, 8),
                 "ff_gemm p=67108859 (largest prime < 2^26), m=n=k=16384, alpha=p-1, beta=1, NN, 1/2/4/8 GPUs"),
}
