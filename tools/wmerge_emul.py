"""Host emulation of one fused pass (csrc/pcf_wmerge.cu) for debugging: k pairwise
non-compacting merges of a node's children with carries, moments kind."""
import numpy as np


def emul_mom(t, v, m2, off, first, C, leaves, nlev):
    lists = []
    for c in range(C):
        a, b = off[first + c], off[first + c + 1]
        lists.append((t[a:b].copy(), v[a:b].copy(), m2[a:b].copy(), v[a], m2[a], float(leaves[c])))
    for _ in range(nlev):
        if len(lists) == 1:
            break
        out = []
        for i in range(0, len(lists), 2):
            if i + 1 >= len(lists):
                out.append(lists[i]); continue
            (ta, va, xa, cva, c2a, na), (tb, vb, xb, cvb, c2b, nb) = lists[i], lists[i + 1]
            n = na + nb; wB = nb / n; wAB = na * nb / n
            T, V, X = [], [], []
            ii = jj = 0
            while ii < len(ta) or jj < len(tb):
                takeA = ii < len(ta) and (jj >= len(tb) or ta[ii] <= tb[jj])
                if takeA:
                    tt = ta[ii]; a_ = va[ii]; b_ = vb[jj - 1] if jj > 0 else cvb
                    x1 = xa[ii]; x2 = xb[jj - 1] if jj > 0 else c2b; ii += 1
                else:
                    tt = tb[jj]; a_ = va[ii - 1] if ii > 0 else cva; b_ = vb[jj]
                    x1 = xa[ii - 1] if ii > 0 else c2a; x2 = xb[jj]; jj += 1
                d = b_ - a_
                T.append(tt); V.append(a_ + d * wB); X.append((x1 + x2) + d * d * wAB)
            d = cvb - cva
            out.append((np.array(T), np.array(V), np.array(X), cva + d * wB, (c2a + c2b) + d * d * wAB, n))
        lists = out
    return lists[0][0], lists[0][1], lists[0][2]
