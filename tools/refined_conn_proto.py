"""Prototype of the closed-form connectivity of a red-refined mesh (pure
Python, small meshes): the child mesh's first-occurrence edge slots
(edge_first) and face mates (slot_mate) from the parent's tables, checked
against the generic star/hash path of the oracle (full tables).  The CUDA
kernel (refine_conn.cu) follows these rules; this file documents and tests
them on CPU.

usage: python tools/refined_conn_proto.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_bind import Oracle, cube5  # noqa: E402

EV = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]   # local edge pairs
FV = [(0, 1, 2), (0, 2, 3), (0, 3, 1), (3, 2, 1)]       # local oriented faces


def ledge(a, b):
    a, b = min(a, b), max(a, b)
    return EV.index((a, b))


def M(a, b):
    return ("m", min(a, b), max(a, b))


C = ("c",)
# refine.cpp:58-61, corner indices 0..3 = i j k l
CH = [
    (0, M(0, 1), M(0, 2), M(0, 3)),
    (1, M(1, 2), M(0, 1), M(1, 3)),
    (2, M(0, 2), M(1, 2), M(2, 3)),
    (3, M(2, 3), M(1, 3), M(0, 3)),
    (M(0, 1), M(0, 2), M(0, 3), C),
    (M(1, 2), M(0, 1), M(1, 3), C),
    (M(0, 2), M(1, 2), M(2, 3), C),
    (M(2, 3), M(1, 3), M(0, 3), C),
    (M(0, 1), M(1, 2), M(0, 2), C),
    (M(0, 2), M(2, 3), M(0, 3), C),
    (M(0, 1), M(0, 3), M(1, 3), C),
    (M(2, 3), M(1, 2), M(1, 3), C),
]


def child_index(t, q, n):
    return t if q == 0 else n + 11 * t + q - 1


def face_excluding(d):
    """local face of a tet that does not contain local vertex d"""
    return {3: 0, 1: 1, 2: 2, 0: 3}[d]


def refined_tables(P, EOS, EF, SM, A0):
    """child edge_first [6 * 12n] and slot_mate [4 * 12n] from the parent:
    P tets [n,4], EOS edge ids per slot [n,6], EF first slot per edge slot
    [6n], SM face mate per slot [4n], A0[e] = (min t with t[0] = smaller
    endpoint, min t with t[0] = larger endpoint) or -1"""
    n = len(P)
    ef = np.full(6 * 12 * n, -1, dtype=np.int64)
    sm = np.full(4 * 12 * n, -2, dtype=np.int64)
    for t in range(n):
        for q in range(12):
            c = child_index(t, q, n)
            ch = CH[q]
            for kk, (u, v) in enumerate(EV):
                A, B = ch[u], ch[v]
                ef[6 * c + kk] = first_edge(t, A, B, P, EOS, EF, SM, A0, n)
            for kf, fv in enumerate(FV):
                S = frozenset(ch[x] for x in fv)
                sm[4 * c + kf] = face_mate(t, q, kf, S, P, SM, n)
    return ef, sm


def first_edge(t, A, B, P, EOS, EF, SM, A0, n):
    corner = [x for x in (A, B) if isinstance(x, int)]
    mids = [x for x in (A, B) if isinstance(x, tuple) and x[0] == "m"]
    if len(corner) == 1:  # half-edge (a, m_ab)
        a = corner[0]
        m = mids[0]
        b = m[1] if m[2] == a else m[2]
        ga, gb = P[t][a], P[t][b]
        e = EOS[t][ledge(a, b)]
        ts = A0[e][0 if ga < gb else 1]
        if ts >= 0:  # C0 of the first parent with vertex 0 = a
            pb = list(P[ts]).index(gb)
            return 6 * ts + (pb - 1)
        t1 = EF[6 * t + ledge(a, b)] // 6
        qa, qb = list(P[t1]).index(ga), list(P[t1]).index(gb)
        p = CH[qa].index(M(qa, qb))
        return 6 * child_index(t1, qa, n) + (p - 1)
    if len(mids) == 2:  # inside a parent face, shared corner a
        (x1, y1), (x2, y2) = mids[0][1:], mids[1][1:]
        a = ({x1, y1} & {x2, y2}).pop()
        b = x1 if y1 == a else y1
        cc = x2 if y2 == a else y2
        d = ({0, 1, 2, 3} - {a, b, cc}).pop()
        kF = face_excluding(d)
        ga, gb, gc = P[t][a], P[t][b], P[t][cc]
        ms = SM[4 * t + kF]
        parents = sorted({t} | ({ms // 4} if ms >= 0 else set()))
        for u in parents:
            if P[u][0] == ga:
                pb, pc = list(P[u]).index(gb), list(P[u]).index(gc)
                return 6 * u + ledge(pb, pc)  # pair (pb, pc) among C0's midpoints at positions pb, pc
        t1 = parents[0]
        qa = list(P[t1]).index(ga)
        qb, qc = list(P[t1]).index(gb), list(P[t1]).index(gc)
        ch = CH[qa]
        p1, p2 = ch.index(M(qa, qb)), ch.index(M(qa, qc))
        return 6 * child_index(t1, qa, n) + ledge(p1, p2)
    # centroid edge (m, c): first in C4 / C5 / C6 of t
    m = mids[0]
    for q in (4, 5, 6):
        if m in CH[q]:
            return 6 * child_index(t, q, n) + ledge(CH[q].index(m), 3)
    raise AssertionError


def face_mate(t, q, kf, S, P, SM, n):
    # a face shared by two children of the same parent
    for q2 in range(12):
        if q2 == q:
            continue
        for kf2, fv in enumerate(FV):
            if frozenset(CH[q2][x] for x in fv) == S:
                return 4 * child_index(t, q2, n) + kf2
    # a sub-triangle of parent face F: mate across F in the other parent
    corners = set()
    for x in S:
        if isinstance(x, int):
            corners.add(x)
        else:
            corners |= {x[1], x[2]}
    assert len(corners) == 3
    d = ({0, 1, 2, 3} - corners).pop()
    kF = face_excluding(d)
    ms = SM[4 * t + kF]
    if ms < 0:
        return -1
    t2 = ms // 4
    loc = {a: list(P[t2]).index(P[t][a]) for a in corners}
    S2 = frozenset(loc[x] if isinstance(x, int) else M(loc[x[1]], loc[x[2]]) for x in S)
    for q2 in range(12):
        for kf2, fv in enumerate(FV):
            if frozenset(CH[q2][x] for x in fv) == S2:
                return 4 * child_index(t2, q2, n) + kf2
    raise AssertionError


def generic_tables(O, m):
    """edge_first and slot_mate of a mesh from the oracle's full tables"""
    _, eos = O.edges(m)
    eos = eos.reshape(-1)
    first = {}
    ef = np.zeros(len(eos), dtype=np.int64)
    for s, e in enumerate(eos):
        first.setdefault(e, s)
        ef[s] = first[e]
    f = O.faces(m)
    fs = f["face_slots"]
    sm = np.zeros(4 * m.ne, dtype=np.int64)
    for a, b in fs:
        sm[a] = b
        if b >= 0:
            sm[b] = a
    return eos.reshape(-1, 6), ef, sm


def a0_table(P, EOS, ned):
    A0 = np.full((ned, 2), -1, dtype=np.int64)
    for t in range(len(P)):
        for k in range(3):  # local pairs (0, x): vertex 0 is an endpoint
            e = EOS[t][k]
            a, b = P[t][0], P[t][k + 1]
            w = 0 if a < b else 1
            if A0[e][w] < 0 or t < A0[e][w]:
                A0[e][w] = t
    return A0


def main():
    O = Oracle()
    for name, m in (("cube5", cube5()), ("kuhn1", O.kuhn(1, 1, 1)), ("kuhn2x1x3", O.kuhn(2, 1, 3, jitter=0.1))):
        for lv in range(3):
            eos, ef, sm = generic_tables(O, m)
            A0 = a0_table(m.tets, eos, int(eos.max()) + 1)
            child = O.refine(m)[0]
            _, ef_c, sm_c = generic_tables(O, child)
            ef_p, sm_p = refined_tables(m.tets, eos, ef, sm, A0)
            ok_e = np.array_equal(ef_p, ef_c)
            ok_f = np.array_equal(sm_p, sm_c)
            print(name, "level", lv, "->", lv + 1, child.ne, "edge_first", ok_e, "slot_mate", ok_f, flush=True)
            if not (ok_e and ok_f):
                bad = np.nonzero(ef_p != ef_c)[0][:5]
                print("  edge mismatches at", bad, ef_p[bad], ef_c[bad])
                bad = np.nonzero(sm_p != sm_c)[0][:5]
                print("  face mismatches at", bad, sm_p[bad], sm_c[bad])
                return 1
            m = child
    return 0


if __name__ == "__main__":
    sys.exit(main())
