"""ctypes bindings of the CPU checkers under oracle/ (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.  Two checkers are bound:

* ``Oracle``   -- oracle/_build/libphfem_oracle.so, the C restatement
                  (oracle/phfem_oracle.c);
* ``RefCtx``   -- oracle/_ref/libphfem_ref.so, the unmodified reference
                  library compiled from its own sources plus the shim
                  oracle/ref_driver.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libphfem_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libphfem_ref.so")

P = C.c_void_p
I64 = C.c_int64


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def build_oracle() -> None:
    """Build oracle/_build (and oracle/_ref where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


# ---------------------------------------------------------------------------
# mesh container shared by all paths


@dataclass
class MeshArrays:
    coords: np.ndarray  # (nC, 3) float64
    tets: np.ndarray  # (nE, 4) int32
    db: np.ndarray  # (nD, 3) int32
    nb: np.ndarray  # (nN, 3) int32
    level: int = 0

    @property
    def nc(self):
        return self.coords.shape[0]

    @property
    def ne(self):
        return self.tets.shape[0]


def cube5() -> MeshArrays:
    """initial_cube_mesh (mesh.cpp:12-32), 1-based tables converted."""
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0],
                       [0, 0, 1], [1, 0, 1], [0, 1, 1], [1, 1, 1]], dtype=np.float64)
    tets = np.array([[1, 2, 3, 5], [5, 8, 6, 2], [7, 3, 8, 5], [4, 8, 3, 2], [8, 3, 2, 5]],
                    dtype=np.int32) - 1
    db = np.array([[7, 8, 5], [5, 8, 6]], dtype=np.int32) - 1
    nb = np.array([[1, 5, 2], [5, 6, 2], [1, 3, 5], [7, 5, 3], [7, 3, 8],
                   [4, 8, 3], [2, 6, 8], [4, 2, 8], [4, 3, 2], [1, 2, 3]], dtype=np.int32) - 1
    return MeshArrays(coords, tets, db, nb, 0)


# ---------------------------------------------------------------------------
# C restatement


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = C.CDLL(path)
        self.L = L
        L.or_last_error.restype = C.c_char_p
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64]
        L.or_uniform.restype = C.c_double
        L.or_uniform.argtypes = [C.c_uint64, C.c_uint64]
        L.or_kuhn_sizes.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32, P]
        L.or_kuhn_mesh.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, C.c_uint32, P, P, P, P]
        L.or_num_edges.restype = I64
        L.or_num_edges.argtypes = [I64, I64, P, P, P]
        L.or_edge_pairs_to_elems.argtypes = [I64, I64, P, P, P]
        L.or_face_table.argtypes = [I64, I64, P, P, I64, P, I64, P, P, P, P, P, P, P, P, P]
        L.or_refine.argtypes = [I64, I64, P, P, I64, P, I64, P, P, P, P, P, P, P]
        L.or_assemble_condense.argtypes = [I64, I64, P, P, I64, P, P, P, P, P, P, P, I64, P] + [P] * 13
        L.or_conn_digests.argtypes = [I64, I64, P, P, P, P]
        L.or_sha256.argtypes = [P, I64, P]
        L.or_entry_scales.argtypes = [I64, I64, P, P, I64, P, P, P, P, P, P, P, I64, P, P, P]
        L.or_pcg.argtypes = [I64, P, P, P, P, P, C.c_double, C.c_double, I64, P]
        L.or_solve_schur.argtypes = [I64, I64, P, P, P, I64] + [P] * 11 + [C.c_double, I64, P, P, P]
        L.or_errors.argtypes = [I64, I64, P, P, P, P, P, P, P, P, P]
        L.or_mesh_diameter.restype = C.c_double
        L.or_mesh_diameter.argtypes = [I64, I64, P, P]
        L.or_tet_rule.argtypes = [C.c_int, P, P]

    def _check(self, rc):
        if rc:
            raise CheckerError(rc, self.L.or_last_error().decode())

    # seeded inputs --------------------------------------------------------
    def uniform(self, seed: int, idx: int) -> float:
        return self.L.or_uniform(seed, idx)

    def kuhn(self, nx, ny, nz, lx=1.0, ly=1.0, lz=1.0, jitter=0.0, seed=2509, dmask=0x3F) -> MeshArrays:
        s = np.zeros(4, dtype=np.int64)
        self.L.or_kuhn_sizes(nx, ny, nz, dmask, _ptr(s))
        nc, ne, nd, nn = (int(v) for v in s)
        coords = np.zeros((nc, 3))
        tets = np.zeros((ne, 4), dtype=np.int32)
        db = np.zeros((nd, 3), dtype=np.int32)
        nb = np.zeros((nn, 3), dtype=np.int32)
        self.L.or_kuhn_mesh(nx, ny, nz, lx, ly, lz, jitter, seed, dmask,
                            _ptr(coords), _ptr(tets), _ptr(db), _ptr(nb))
        return MeshArrays(coords, tets, db, nb, 0)

    # connectivity ---------------------------------------------------------
    def edges(self, m: MeshArrays):
        eos = np.zeros((m.ne, 6), dtype=np.int32)
        en = np.zeros((6 * m.ne + 1, 2), dtype=np.int32)
        ned = self.L.or_num_edges(m.nc, m.ne, _ptr(m.tets), _ptr(eos), _ptr(en))
        return en[:ned].copy(), eos

    def e2t(self, m: MeshArrays):
        keys = np.zeros(12 * m.ne, dtype=np.uint64)
        elems = np.zeros(12 * m.ne, dtype=np.int32)
        self._check(self.L.or_edge_pairs_to_elems(m.nc, m.ne, _ptr(m.tets), _ptr(keys), _ptr(elems)))
        return keys, elems

    def faces(self, m: MeshArrays) -> dict:
        cap = 4 * m.ne
        out = dict(
            faces=np.zeros((cap, 3), dtype=np.int32),
            face_of_slot=np.zeros(cap, dtype=np.int32),
            sigma=np.zeros(cap, dtype=np.int8),
            face_slots=np.zeros((cap, 2), dtype=np.int64),
            face_class=np.zeros(cap, dtype=np.uint8),
            mrow=np.zeros(cap, dtype=np.int32),
            area=np.zeros(cap, dtype=np.float64),
        )
        counts = np.zeros(5, dtype=np.int64)
        self._check(self.L.or_face_table(
            m.nc, m.ne, _ptr(m.tets), _ptr(m.coords), len(m.db), _ptr(m.db), len(m.nb), _ptr(m.nb),
            _ptr(out["faces"]), _ptr(out["face_of_slot"]), _ptr(out["sigma"]), _ptr(out["face_slots"]),
            _ptr(out["face_class"]), _ptr(out["mrow"]), _ptr(out["area"]), _ptr(counts)))
        nf = int(counts[0])
        for k in ("faces", "face_slots", "face_class", "mrow", "area"):
            out[k] = out[k][:nf].copy()
        out.update(nf=nf, n_interior=int(counts[1]), n_dirichlet=int(counts[2]),
                   n_neumann=int(counts[3]), l=int(counts[4]))
        return out

    def refine(self, m: MeshArrays):
        en, _ = self.edges(m)
        ned = len(en)
        coords = np.zeros((m.nc + ned + m.ne, 3))
        tets = np.zeros((12 * m.ne, 4), dtype=np.int32)
        db = np.zeros((4 * len(m.db), 3), dtype=np.int32)
        nb = np.zeros((4 * len(m.nb), 3), dtype=np.int32)
        mid = np.zeros(ned, dtype=np.int32)
        cen = np.zeros(m.ne, dtype=np.int32)
        self._check(self.L.or_refine(m.nc, m.ne, _ptr(m.coords), _ptr(m.tets), len(m.db), _ptr(m.db),
                                     len(m.nb), _ptr(m.nb), _ptr(coords), _ptr(tets), _ptr(db), _ptr(nb),
                                     _ptr(mid), _ptr(cen)))
        return MeshArrays(coords, tets, db, nb, m.level + 1), mid, cen

    # assembly + condensation ---------------------------------------------
    class _Prob(C.Structure):
        _fields_ = [("kind", C.c_int), ("c", C.c_double), ("a_elem", P), ("a_diag", P)]

    def _prob(self, kind, c, a_elem, a_diag):
        return self._Prob(kind, c, _ptr(a_elem), _ptr(a_diag))

    def assemble(self, m: MeshArrays, ft: dict, kind=0, c=1.0, a_elem=None, a_diag=None,
                 schur=True, with_c=True) -> dict:
        ne, l = m.ne, ft["l"]
        pr = self._prob(kind, c, a_elem, a_diag)
        out = dict(a_blocks=np.zeros((ne, 4, 4)), slot_coef=np.zeros((ne, 4)),
                   slot_mrow=np.zeros((ne, 4), dtype=np.int32), rhs=np.zeros(4 * ne), bd=np.zeros(l))
        if with_c:
            out.update(c_rowptr=np.zeros(l + 1, dtype=np.int64), c_col=np.zeros(12 * ne + 1, dtype=np.int32),
                       c_val=np.zeros(12 * ne + 1))
        if schur:
            out.update(s_rowptr=np.zeros(l + 1, dtype=np.int64), s_col=np.zeros(16 * ne + 1, dtype=np.int32),
                       s_val=np.zeros(16 * ne + 1), rhs_neg=np.zeros(l))
        nnz = np.zeros(1, dtype=np.int64)
        g = out.get
        self._check(self.L.or_assemble_condense(
            m.nc, ne, _ptr(m.coords), _ptr(m.tets), ft["nf"], _ptr(ft["faces"]), _ptr(ft["face_of_slot"]),
            _ptr(ft["sigma"]), _ptr(ft["face_slots"]), _ptr(ft["face_class"]), _ptr(ft["mrow"]),
            _ptr(ft["area"]), l, C.byref(pr), _ptr(out["a_blocks"]), _ptr(out["slot_coef"]),
            _ptr(out["slot_mrow"]), _ptr(out["rhs"]), _ptr(out["bd"]), _ptr(g("c_rowptr")), _ptr(g("c_col")),
            _ptr(g("c_val")), _ptr(g("s_rowptr")), _ptr(g("s_col")), _ptr(g("s_val")), _ptr(g("rhs_neg")),
            _ptr(nnz)))
        if with_c:
            cn = int(out["c_rowptr"][-1])
            out["c_col"] = out["c_col"][:cn].copy()
            out["c_val"] = out["c_val"][:cn].copy()
        if schur:
            sn = int(nnz[0])
            out["s_col"] = out["s_col"][:sn].copy()
            out["s_val"] = out["s_val"][:sn].copy()
        return out

    def solve(self, m: MeshArrays, sys: dict, kind=0, c=1.0, a_elem=None, a_diag=None, tol=1e-10,
              max_iter=-1):
        pr = self._prob(kind, c, a_elem, a_diag)
        l = len(sys["bd"])
        u = np.zeros(4 * m.ne)
        lam = np.zeros(l)
        st = np.zeros(3)
        self._check(self.L.or_solve_schur(
            m.nc, m.ne, _ptr(m.coords), _ptr(m.tets), C.byref(pr), l, _ptr(sys["slot_coef"]),
            _ptr(sys["slot_mrow"]), _ptr(sys["rhs"]), _ptr(sys["bd"]), _ptr(sys["c_rowptr"]),
            _ptr(sys["c_col"]), _ptr(sys["c_val"]), _ptr(sys["s_rowptr"]), _ptr(sys["s_col"]),
            _ptr(sys["s_val"]), _ptr(sys["rhs_neg"]), tol, max_iter, _ptr(u), _ptr(lam), _ptr(st)))
        return u, lam, dict(iterations=int(st[0]), residual=st[1], constraint_residual=st[2])

    DIGEST_KEYS = ("edge_nodes", "edge_of_slot", "faces", "face_of_slot", "sigma", "face_slots", "area",
                   "face_class", "mrow")

    def conn_digests(self, m: MeshArrays) -> dict:
        """streaming SHA-256 digests of the connectivity arrays
        (or_conn_digests; all-Dirichlet meshes)"""
        d = np.zeros(32 * len(self.DIGEST_KEYS), dtype=np.uint8)
        c = np.zeros(2, dtype=np.int64)
        self._check(self.L.or_conn_digests(m.nc, m.ne, _ptr(m.tets), _ptr(m.coords), _ptr(d), _ptr(c)))
        out = {k: bytes(d[32 * i:32 * i + 32]).hex() for i, k in enumerate(self.DIGEST_KEYS)}
        out.update(ned=int(c[0]), nf=int(c[1]))
        return out

    def sha256(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a)
        d = np.zeros(32, dtype=np.uint8)
        self.L.or_sha256(_ptr(a), a.nbytes, _ptr(d))
        return bytes(d).hex()

    def entry_scales(self, m: MeshArrays, ft: dict, kind=0, c=1.0, a_elem=None, a_diag=None):
        """componentwise magnitudes of B_T and rhs_neg (or_entry_scales)"""
        pr = self._prob(kind, c, a_elem, a_diag)
        rs = np.zeros(4 * m.ne)
        ns = np.zeros(ft["l"])
        self._check(self.L.or_entry_scales(
            m.nc, m.ne, _ptr(m.coords), _ptr(m.tets), ft["nf"], _ptr(ft["faces"]), _ptr(ft["face_of_slot"]),
            _ptr(ft["sigma"]), _ptr(ft["face_slots"]), _ptr(ft["face_class"]), _ptr(ft["mrow"]),
            _ptr(ft["area"]), ft["l"], C.byref(pr), _ptr(rs), _ptr(ns)))
        return rs, ns

    def solve_raw(self, m: MeshArrays, sys: dict, kind=0, c=1.0, a_elem=None, a_diag=None, tol=1e-10,
                  max_iter=-1):
        """or_solve_schur without raising: U, Lambda and the stats are filled
        before verify_solution decides (solver.cpp:44-76), so a refused solve
        still yields its iterates.  Returns (u, lambda, stats, rc, message)."""
        pr = self._prob(kind, c, a_elem, a_diag)
        l = len(sys["bd"])
        u = np.zeros(4 * m.ne)
        lam = np.zeros(l)
        st = np.zeros(3)
        rc = self.L.or_solve_schur(
            m.nc, m.ne, _ptr(m.coords), _ptr(m.tets), C.byref(pr), l, _ptr(sys["slot_coef"]),
            _ptr(sys["slot_mrow"]), _ptr(sys["rhs"]), _ptr(sys["bd"]), _ptr(sys["c_rowptr"]),
            _ptr(sys["c_col"]), _ptr(sys["c_val"]), _ptr(sys["s_rowptr"]), _ptr(sys["s_col"]),
            _ptr(sys["s_val"]), _ptr(sys["rhs_neg"]), tol, max_iter, _ptr(u), _ptr(lam), _ptr(st))
        msg = self.L.or_last_error().decode() if rc else ""
        return u, lam, dict(iterations=int(st[0]), residual=st[1], constraint_residual=st[2]), rc, msg

    def pcg(self, sys: dict, tol=1e-10, abs_tol=0.0, max_iter=-1):
        l = len(sys["rhs_neg"])
        x = np.zeros(l)
        res = np.zeros(3)
        self._check(self.L.or_pcg(l, _ptr(sys["s_rowptr"]), _ptr(sys["s_col"]), _ptr(sys["s_val"]),
                                  _ptr(sys["rhs_neg"]), _ptr(x), tol, abs_tol, max_iter, _ptr(res)))
        return x, res

    def errors(self, m: MeshArrays, ft: dict, u, lam, kind=0, c=1.0, a_elem=None, a_diag=None):
        pr = self._prob(kind, c, a_elem, a_diag)
        out = np.zeros(3)
        self._check(self.L.or_errors(m.nc, m.ne, _ptr(m.coords), _ptr(m.tets), _ptr(ft["face_of_slot"]),
                                     _ptr(ft["sigma"]), _ptr(ft["mrow"]), C.byref(pr), _ptr(u), _ptr(lam),
                                     _ptr(out)))
        return out

    def diameter(self, m: MeshArrays) -> float:
        return self.L.or_mesh_diameter(m.nc, m.ne, _ptr(m.coords), _ptr(m.tets))

    def tet_rule(self, degree):
        n = (degree + 4) // 2
        lam = np.zeros((n ** 3, 4))
        w = np.zeros(n ** 3)
        self.L.or_tet_rule(degree, _ptr(lam), _ptr(w))
        return lam, w


# ---------------------------------------------------------------------------
# the reference itself (oracle/_ref)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefLib:
    _inst = None

    def __init__(self, path: str = REF_SO):
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_ctx_new.restype = P
        L.ref_ctx_new.argtypes = [P, I64, P, I64, P, I64, P, I64, C.c_int]
        L.ref_ctx_new_cube.restype = P
        L.ref_ctx_free.argtypes = [P]
        L.ref_mesh_sizes.argtypes = [P, P]
        L.ref_mesh_get.argtypes = [P, P, P, P, P]
        L.ref_connectivity.argtypes = [P, P]
        L.ref_num_edges.argtypes = [P, P]
        L.ref_conn_counts.argtypes = [P, P]
        L.ref_get_edges.argtypes = [P, P, P]
        L.ref_e2t_size.restype = I64
        L.ref_e2t_size.argtypes = [P]
        L.ref_get_e2t.argtypes = [P, P, P]
        L.ref_get_faces.argtypes = [P, P, P, P, P, P, P, P]
        L.ref_refine.argtypes = [P, P]
        L.ref_get_refinement_map.argtypes = [P, P, P]
        L.ref_set_coefficients.argtypes = [P, P, P, C.c_double]
        L.ref_assemble.argtypes = [P, C.c_int, P]
        L.ref_system_sizes.argtypes = [P, P]
        L.ref_get_system.argtypes = [P] + [P] * 8
        L.ref_build_schur.argtypes = [P, C.c_int, P]
        L.ref_schur_nnz.restype = I64
        L.ref_schur_nnz.argtypes = [P]
        L.ref_get_schur.argtypes = [P, P, P, P, P]
        L.ref_cg_prefix.argtypes = [P, I64, C.c_double, P, P]
        L.ref_solve.argtypes = [P, C.c_char_p, C.c_int, C.c_double, I64, P]
        L.ref_get_solution.argtypes = [P, P, P]
        L.ref_errors.argtypes = [P, P]

    @classmethod
    def get(cls):
        if cls._inst is None:
            cls._inst = RefLib()
        return cls._inst


class RefCtx:
    """One reference Mesh (+ connectivity, system, solution) in oracle/_ref."""

    def __init__(self, m: MeshArrays | None = None):
        self.R = RefLib.get()
        L = self.R.L
        if m is None:
            self.h = L.ref_ctx_new_cube()
        else:
            self.h = L.ref_ctx_new(_ptr(np.ascontiguousarray(m.coords)), m.nc, _ptr(np.ascontiguousarray(m.tets)),
                                   m.ne, _ptr(np.ascontiguousarray(m.db)), len(m.db),
                                   _ptr(np.ascontiguousarray(m.nb)), len(m.nb), m.level)

    def __del__(self):
        try:
            self.R.L.ref_ctx_free(self.h)
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            raise CheckerError(rc, self.R.L.ref_last_error().decode())

    def mesh(self) -> MeshArrays:
        s = np.zeros(5, dtype=np.int64)
        self.R.L.ref_mesh_sizes(self.h, _ptr(s))
        nc, ne, nd, nn, lv = (int(v) for v in s)
        m = MeshArrays(np.zeros((nc, 3)), np.zeros((ne, 4), dtype=np.int32), np.zeros((nd, 3), dtype=np.int32),
                       np.zeros((nn, 3), dtype=np.int32), lv)
        self.R.L.ref_mesh_get(self.h, _ptr(m.coords), _ptr(m.tets), _ptr(m.db), _ptr(m.nb))
        return m

    def connectivity(self):
        t = np.zeros(4)
        self._check(self.R.L.ref_connectivity(self.h, _ptr(t)))
        return t

    def num_edges(self):
        t = np.zeros(1)
        self._check(self.R.L.ref_num_edges(self.h, _ptr(t)))
        return float(t[0])

    def counts(self):
        c = np.zeros(6, dtype=np.int64)
        self.R.L.ref_conn_counts(self.h, _ptr(c))
        return dict(ned=int(c[0]), nf=int(c[1]), n_interior=int(c[2]), n_dirichlet=int(c[3]),
                    n_neumann=int(c[4]), l=int(c[5]))

    def edges(self):
        ne = self.mesh().ne
        c = self.counts()
        en = np.zeros((c["ned"], 2), dtype=np.int32)
        eos = np.zeros((ne, 6), dtype=np.int32)
        self.R.L.ref_get_edges(self.h, _ptr(en), _ptr(eos))
        return en, eos

    def e2t(self):
        n = self.R.L.ref_e2t_size(self.h)
        keys = np.zeros(n, dtype=np.uint64)
        elems = np.zeros(n, dtype=np.int32)
        self.R.L.ref_get_e2t(self.h, _ptr(keys), _ptr(elems))
        return keys, elems

    def faces(self) -> dict:
        ne = self.mesh().ne
        c = self.counts()
        nf = c["nf"]
        out = dict(faces=np.zeros((nf, 3), dtype=np.int32), face_of_slot=np.zeros(4 * ne, dtype=np.int32),
                   sigma=np.zeros(4 * ne, dtype=np.int8), face_slots=np.zeros((nf, 2), dtype=np.int64),
                   face_class=np.zeros(nf, dtype=np.uint8), mrow=np.zeros(nf, dtype=np.int32),
                   area=np.zeros(nf))
        self.R.L.ref_get_faces(self.h, _ptr(out["faces"]), _ptr(out["face_of_slot"]), _ptr(out["sigma"]),
                               _ptr(out["face_slots"]), _ptr(out["face_class"]), _ptr(out["mrow"]),
                               _ptr(out["area"]))
        out.update(nf=nf, n_interior=c["n_interior"], n_dirichlet=c["n_dirichlet"],
                   n_neumann=c["n_neumann"], l=c["l"])
        return out

    def refine(self):
        parent = self.mesh()
        if self.counts()["ned"] < 0:
            self.num_edges()
        ned = self.counts()["ned"]
        t = np.zeros(1)
        self._check(self.R.L.ref_refine(self.h, _ptr(t)))
        mid = np.zeros(ned, dtype=np.int32)
        cen = np.zeros(parent.ne, dtype=np.int32)
        self.R.L.ref_get_refinement_map(self.h, _ptr(mid), _ptr(cen))
        return mid, cen, float(t[0])

    def set_coefficients(self, a_elem=None, a_diag=None, c=1.0):
        self.R.L.ref_set_coefficients(self.h, _ptr(a_elem), _ptr(a_diag), c)

    def assemble(self, kind=0):
        t = np.zeros(1)
        self._check(self.R.L.ref_assemble(self.h, kind, _ptr(t)))
        s = np.zeros(3, dtype=np.int64)
        self.R.L.ref_system_sizes(self.h, _ptr(s))
        n, l, cnnz = (int(v) for v in s)
        ne = n // 4
        out = dict(a_blocks=np.zeros((ne, 4, 4)), slot_coef=np.zeros((ne, 4)),
                   slot_mrow=np.zeros((ne, 4), dtype=np.int32), rhs=np.zeros(n), bd=np.zeros(l),
                   c_rowptr=np.zeros(l + 1, dtype=np.int64), c_col=np.zeros(cnnz, dtype=np.int32),
                   c_val=np.zeros(cnnz), t_assemble=float(t[0]))
        self.R.L.ref_get_system(self.h, _ptr(out["a_blocks"]), _ptr(out["slot_coef"]), _ptr(out["slot_mrow"]),
                                _ptr(out["rhs"]), _ptr(out["bd"]), _ptr(out["c_rowptr"]), _ptr(out["c_col"]),
                                _ptr(out["c_val"]))
        return out

    def build_schur(self, workers=1):
        t = np.zeros(1)
        self._check(self.R.L.ref_build_schur(self.h, workers, _ptr(t)))
        nnz = self.R.L.ref_schur_nnz(self.h)
        l = self.counts()["l"]
        out = dict(s_rowptr=np.zeros(l + 1, dtype=np.int64), s_col=np.zeros(nnz, dtype=np.int32),
                   s_val=np.zeros(nnz), rhs_neg=np.zeros(l), t_schur=float(t[0]))
        self.R.L.ref_get_schur(self.h, _ptr(out["s_rowptr"]), _ptr(out["s_col"]), _ptr(out["s_val"]),
                               _ptr(out["rhs_neg"]))
        return out

    def cg_prefix(self, iters, tol=1e-10):
        sec = np.zeros(1)
        done = np.zeros(1, dtype=np.int64)
        self._check(self.R.L.ref_cg_prefix(self.h, iters, tol, _ptr(sec), _ptr(done)))
        return float(sec[0]), int(done[0])

    def solve(self, method="schur", workers=1, tol=1e-10, max_iter=-1):
        st = np.zeros(4)
        self._check(self.R.L.ref_solve(self.h, method.encode(), workers, tol, max_iter, _ptr(st)))
        ne = self.mesh().ne
        l = self.counts()["l"]
        u = np.zeros(4 * ne)
        lam = np.zeros(l)
        self.R.L.ref_get_solution(self.h, _ptr(u), _ptr(lam))
        return u, lam, dict(iterations=int(st[0]), residual=st[1], constraint_residual=st[2], seconds=st[3])

    def errors(self):
        out = np.zeros(3)
        self._check(self.R.L.ref_errors(self.h, _ptr(out)))
        return out
