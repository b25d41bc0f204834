"""Interaction counts of an adaptive tree by dual-tree traversal (SURVEY 8(f)-4 study, not product
code): leaves = boxes with n_src + n_fld <= m (or depth D), traversal from all level-2 pairs:
S2L if max(|dr|, |dz|) >= h_T + h_S, P2P if both leaves, else split the leaf-free side (both
when of equal size).  With m = 0 it reproduces Algorithm 1's lists exactly (C2: 31,920 S2L box
pairs, 2,284,652 near pairs).   python tools/dtt_counts.py C5 10 64"""
import sys, numpy as np, time
sys.path.insert(0, '/root/repo')
from paper_2301_01179_b200.inputs import CONFIGS
name = sys.argv[1]; D = int(sys.argv[2]); m = int(sys.argv[3])
pr = CONFIGS[name]()
L, z0 = pr.L, pr.z0
def boxes(r, z, l):
    nb = 1 << l
    return np.minimum((r * nb / L).astype(np.int64), nb-1), np.minimum(((z - z0) * nb / L).astype(np.int64), nb-1)
# counts per level (dense)
ns, nt = {}, {}
for l in range(2, D+1):
    nb = 1 << l
    a = np.zeros((nb, nb), np.int64); i, j = boxes(pr.sr, pr.sz, l); np.add.at(a, (i, j), 1); ns[l] = a
    b = np.zeros((nb, nb), np.int64); i, j = boxes(pr.fr, pr.fz, l); np.add.at(b, (i, j), 1); nt[l] = b
leaf = {}; intree = {}
for l in range(2, D+1):
    nb = 1 << l
    if l == 2: it = np.ones((nb, nb), bool)
    else:
        par = intree[l-1] & ~leaf[l-1]
        it = np.repeat(np.repeat(par, 2, 0), 2, 1)
    intree[l] = it
    leaf[l] = it & ((l == D) | (ns[l] + nt[l] <= m))
# frontier: arrays of (lt, it, jt, ls, is, js)
T = np.argwhere(nt[2] > 0); S = np.argwhere(ns[2] > 0)
fr = np.array([(2, a, b, 2, c, d) for a, b in T for c, d in S], np.int64)
s2l_same = s2l_mixed = 0; p2p_pairs = 0; p2p_boxpairs = 0
mixed_geoms = set()
t0 = time.time()
while len(fr):
    lt, it_, jt, ls, is_, js = fr.T
    ht = L / (1 << lt); hs = L / (1 << ls)
    rt = (it_ + 0.5) * ht; zt = (jt + 0.5) * ht; rs = (is_ + 0.5) * hs; zs = (js + 0.5) * hs
    mac = np.maximum(np.abs(rt - rs), np.abs(zt - zs)) >= ht + hs
    tleaf = np.array([leaf[a][b, c] for a, b, c in zip(lt, it_, jt)], bool) if len(fr) < 200000 else None
    if tleaf is None:
        tleaf = np.zeros(len(fr), bool); sleaf = np.zeros(len(fr), bool)
        for l in range(2, D+1):
            sel = lt == l; tleaf[sel] = leaf[l][it_[sel], jt[sel]]
            sel = ls == l; sleaf[sel] = leaf[l][is_[sel], js[sel]]
    else:
        sleaf = np.array([leaf[a][b, c] for a, b, c in zip(ls, is_, js)], bool)
    same = lt == ls
    s2l_same += int((mac & same).sum()); s2l_mixed += int((mac & ~same).sum())
    for row in fr[mac & ~same][:0]: pass
    pp = ~mac & tleaf & sleaf
    p2p_boxpairs += int(pp.sum())
    for l in range(2, D+1):
        pass
    # point pairs
    if pp.any():
        ntv = np.array([nt[a][b, c] for a, b, c in zip(lt[pp], it_[pp], jt[pp])]) if pp.sum() < 100000 else None
        if ntv is None:
            ntv = np.zeros(pp.sum(), np.int64); nsv = np.zeros(pp.sum(), np.int64)
            LT, IT, JT, LS, IS, JS = lt[pp], it_[pp], jt[pp], ls[pp], is_[pp], js[pp]
            for l in range(2, D+1):
                sel = LT == l; ntv[sel] = nt[l][IT[sel], JT[sel]]
                sel = LS == l; nsv[sel] = ns[l][IS[sel], JS[sel]]
        else:
            nsv = np.array([ns[a][b, c] for a, b, c in zip(ls[pp], is_[pp], js[pp])])
        p2p_pairs += int((ntv * nsv).sum())
    rest = ~mac & ~pp
    new = []
    R = fr[rest]; tl_ = tleaf[rest]; sl_ = sleaf[rest]
    # split S if T leaf; split T if S leaf; else split both
    for mode, sel in (('S', tl_), ('T', ~tl_ & sl_), ('B', ~tl_ & ~sl_)):
        X = R[sel]
        if not len(X): continue
        lt, it_, jt, ls, is_, js = X.T
        if mode in ('T', 'B'):
            lt2 = np.repeat(lt + 1, 4); it2 = np.repeat(2 * it_, 4) + np.tile([0, 1, 0, 1], len(X)); jt2 = np.repeat(2 * jt, 4) + np.tile([0, 0, 1, 1], len(X))
            rest_s = [np.repeat(a, 4) for a in (ls, is_, js)]
            Y = np.stack([lt2, it2, jt2] + rest_s, 1)
        else:
            Y = X
        if mode in ('S', 'B'):
            lt, it_, jt, ls, is_, js = Y.T
            ls2 = np.repeat(ls + 1, 4); is2 = np.repeat(2 * is_, 4) + np.tile([0, 1, 0, 1], len(Y)); js2 = np.repeat(2 * js, 4) + np.tile([0, 0, 1, 1], len(Y))
            Y = np.stack([np.repeat(lt, 4), np.repeat(it_, 4), np.repeat(jt, 4), ls2, is2, js2], 1)
        # keep nonempty
        keep = np.zeros(len(Y), bool)
        lt, it_, jt, ls, is_, js = Y.T
        for l in range(2, D+1):
            for l2 in range(2, D+1):
                sel = (lt == l) & (ls == l2)
                if sel.any(): keep[sel] = (nt[l][it_[sel], jt[sel]] > 0) & (ns[l2][is_[sel], js[sel]] > 0)
        new.append(Y[keep])
    fr = np.concatenate(new) if new else np.zeros((0, 6), np.int64)
print(name, 'D', D, 'm', m, 's2l same', s2l_same, 'mixed', s2l_mixed, 'p2p boxpairs', p2p_boxpairs, 'point pairs', p2p_pairs, 'time', round(time.time()-t0,1))
