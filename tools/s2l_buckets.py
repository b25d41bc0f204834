"""C5 S2L batches by fill (study, not product code): the pairs of Algorithm 1's interaction lists
 bucketed by (inner column, class, in/outward) as `s2l_count_kernel` does, cut into
batches of JT = 12.  Prints the tail-size histogram and the share of active column groups (4 pairs
each): the quantity the S2L phase time follows.   python tools/s2l_buckets.py"""
import sys
from collections import Counter
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2301_01179_b200.inputs import surface_sources

sr, sz = surface_sources(4194304)[:2]
L, z0, D, JT, C = 2.0, 0.0, 10, 12, 4
cnt = Counter()
tot = 0
for l in range(2, D + 1):
    nb = 1 << l
    i = np.minimum((sr * nb / L).astype(np.int64), nb - 1)
    j = np.minimum(((sz - z0) * nb / L).astype(np.int64), nb - 1)
    occ = np.zeros((nb, nb), bool)
    occ[i, j] = True
    for si, sj in np.argwhere(occ):
        pi, pj = si // 2, sj // 2
        for ti in range(max(0, 2 * (pi - 1)), min(nb, 2 * (pi + 2))):
            for tj in range(max(0, 2 * (pj - 1)), min(nb, 2 * (pj + 2))):
                di, dj = ti - si, tj - sj
                if max(abs(di), abs(dj)) < 2:
                    continue
                cnt[(min(si, ti), abs(di), abs(dj), int(ti < si) if di else 0)] += 1
                tot += 1
sizes = np.array(list(cnt.values()))
nbatch = int(np.ceil(sizes / JT).sum())
full = int((sizes // JT).sum())
tails = sizes % JT
groups = full * (JT // C) + int(np.ceil(tails / C).sum())
print(f"pairs {tot}  station keys {len(sizes)}  batches {nbatch}  full {full}  pair-slot fill {tot / (nbatch * JT):.3f}")
print("tail sizes 0..11:", np.bincount(tails, minlength=JT).tolist())
print(f"active column groups {groups} of {nbatch * (JT // C)} ({groups / (nbatch * (JT // C)):.3f}); fill inside them {tot / (groups * C):.3f}")
