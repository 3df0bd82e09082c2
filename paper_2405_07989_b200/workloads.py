"""Seeded synthetic workloads (instances) shared by tests, bench.py and smoke().

This module holds NO arithmetic of the method: only instance definitions (n, generators)
and a seeded sampler of random instances.  Both the CUDA path and the oracle receive the
same instances from here.  Recipes are stated in DESIGN.md ("Input recipe").

Config names follow BASELINE.json `configs` / SURVEY.md Sec. 8(d):
  C1   McNugget <6,9,20>, n=1000                                  (configs[0])
  C2   d=5 <11,13,17,19,23>, n=2000                               (configs[1])
  C2L  same generators, n=12000  (materialise at HBM-roofline size, 8.25 GB of u16 rows)
  C2XL same generators, n=16000  (26 GB of u16 rows)
  C3   d=8, sorted(random.Random(240507989).sample(range(10,41),8)), n=4275, |Z|~1e11 (configs[2])
  C4   = C3 with the length histogram, 1/2/4/8 GPUs                  (configs[3])
  C5   skewed/non-minimal <1,1,2,997,1000>, n=20000                  (configs[4])
"""
from __future__ import annotations

import random
from dataclasses import dataclass
from typing import List, Tuple


@dataclass(frozen=True)
class Instance:
    name: str
    n: int
    gens: Tuple[int, ...]

    @property
    def d(self) -> int:
        return len(self.gens)


def c3_generators() -> Tuple[int, ...]:
    """The C3/C4 generator draw (seed 240507989)."""
    return tuple(sorted(random.Random(240507989).sample(range(10, 41), 8)))


C1 = Instance("C1", 1000, (6, 9, 20))
C2 = Instance("C2", 2000, (11, 13, 17, 19, 23))
C2L = Instance("C2L", 12000, (11, 13, 17, 19, 23))
C2XL = Instance("C2XL", 16000, (11, 13, 17, 19, 23))
C3 = Instance("C3", 4275, c3_generators())
C4 = Instance("C4", 4275, c3_generators())
C5 = Instance("C5", 20000, (1, 1, 2, 997, 1000))
C5Q = Instance("C5Q", 10000, (1, 1, 2, 997, 1000))  # quick variant
# C2's shape with a non-coprime last pair (gcd(18, 24) = 6: 5 of 6 level-L nodes have no
# factorization) -- exercises the common-divisor skip of the materialise kernel (NEXT-3)
C2CD = Instance("C2CD", 12000, (11, 13, 17, 18, 24))
# ... and with the last THREE generators sharing 6 (gcd(12, 18, 24)): 5 of 6 level-(L-1)
# subtrees (runs) are dead too -- the k >= 3 skip of the generic ascend (NEXT-3)
C3CD = Instance("C3CD", 12000, (11, 13, 12, 18, 24))

CONFIGS = {i.name: i for i in (C1, C2, C2L, C2XL, C3, C4, C5, C5Q)}

# PAPER.md Table 1: cumulative generator prefixes of (13,37,38,40,41,42,43)
TABLE1_GENS = (13, 37, 38, 40, 41, 42, 43)


def table1_instances() -> List[Instance]:
    rows = [
        (3, [1000, 20000, 45000, 70000, 150000, 225000, 300000, 500000]),
        (4, [1000, 5000, 9000, 13000, 17000, 20000, 23000, 27000, 45000]),
        (5, [1000, 3000, 5000, 7000, 9000]),
        (6, [1000, 1500, 2000, 3000]),
        (7, [1000, 1500, 2000]),
    ]
    out = []
    for d, ns in rows:
        for n in ns:
            out.append(Instance("T1_d%d_n%d" % (d, n), n, TABLE1_GENS[:d]))
    return out


def random_instances(count: int, seed: int = 0, d_max: int = 5, g_max: int = 50,
                     n_max: int = 2000, d_min: int = 1) -> List[Instance]:
    """SPEC.md:333-334 style random suite: d <= d_max, 1 <= g_i <= g_max (duplicates,
    non-coprime and unsorted allowed), 0 <= n <= n_max.  Seeded, deterministic."""
    rng = random.Random(seed)
    out = []
    for i in range(count):
        d = rng.randint(d_min, d_max)
        gens = tuple(rng.randint(1, g_max) for _ in range(d))
        n = rng.randint(0, n_max)
        out.append(Instance("rand%d_s%d" % (i, seed), n, gens))
    return out
