"""Python host binding of libphfem.so (the B200 phfem hot path).

A thin ctypes mirror of the reference C ABI (/root/reference/proj/include/
phfem.h) and of include/phfem_ext.h: the same handles, calls, status codes
and error behaviour, surfaced as Python objects.  There is no Python or CPU
compute path here: every numerical call runs the CUDA kernels inside
libphfem.so, and importing this module fails loudly when the library has not
been built (``python __graft_entry__.py build`` or ``make -C
paper_2509_11133_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PHFEM_LIB selects another build of the same library (experiment builds)
LIB_PATH = os.environ.get("PHFEM_LIB") or os.path.join(HERE, "lib", "libphfem.so")

OK, ERR_ARGUMENT, ERR_MESH, ERR_SOLVER, ERR_IO = 0, 1, 2, 3, 4
PROBLEM_MANUFACTURED, PROBLEM_LINEAR, PROBLEM_ZERO = 0, 1, 2
PROBLEM_SIN3, PROBLEM_EXPCOS, PROBLEM_POLYSIN = 3, 4, 5


class PhfemError(RuntimeError):
    code = -1

    def __init__(self, msg: str):
        super().__init__(msg)
        self.msg = msg


class ArgumentError(PhfemError):
    code = ERR_ARGUMENT


class MeshError(PhfemError):
    code = ERR_MESH


class SolverError(PhfemError):
    code = ERR_SOLVER


class IoError(PhfemError):
    code = ERR_IO


_ERRORS = {ERR_ARGUMENT: ArgumentError, ERR_MESH: MeshError, ERR_SOLVER: SolverError, ERR_IO: IoError}

P = C.c_void_p
I64 = C.c_int64
PP = C.POINTER(C.c_void_p)


class RefineTimes(C.Structure):
    _fields_ = [("t_numedges", C.c_double), ("t_edge2tetra", C.c_double), ("t_faceup", C.c_double),
                ("t_redrefine", C.c_double)]


class StageMs(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("star", "groups", "number", "classify", "assemble", "refine", "total",
                                          "assemble_kernel")]


_lib = None


def lib():
    """Load libphfem.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libphfem.so not built at {LIB_PATH}; run `python __graft_entry__.py build`")
    L = C.CDLL(LIB_PATH)
    L.phfem_last_error.restype = C.c_char_p
    sig = {
        "phfem_mesh_create_cube": [PP],
        "phfem_mesh_read": [C.c_char_p, PP],
        "phfem_mesh_write": [P, C.c_char_p],
        "phfem_mesh_refine": [P, P],
        "phfem_mesh_counts": [P, P, P, P, P, P],
        "phfem_mesh_system_dims": [P, P, P],
        "phfem_mesh_diameter": [P, P],
        "phfem_mesh_dump_connectivity": [P, C.c_char_p, C.c_char_p],
        "phfem_solve": [P, C.c_int, C.c_char_p, C.c_int, C.c_double, PP],
        "phfem_solution_values": [P, P, P, P, P],
        "phfem_solution_stats_json": [P, P],
        "phfem_solution_errors": [P, P, P],
        "phfem_solution_write": [P, C.c_char_p, C.c_char_p],
        "phfem_export_vtk": [P, P, C.c_char_p, C.c_int],
        "phfem_export_multiplier_vtk": [P, C.c_char_p],
        "phfem_dump_system": [P, C.c_int, C.c_char_p],
        "phfem_mesh_create_from_arrays": [P, I64, P, I64, P, I64, P, I64, C.c_int, PP],
        "phfem_mesh_create_from_arrays_async": [P, I64, P, I64, P, I64, P, I64, C.c_int, PP],
        "phfem_mesh_create_kuhn": [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_uint64, C.c_uint32, PP],
        "phfem_mesh_sizes": [P, P],
        "phfem_mesh_get_arrays": [P, P, P, P, P],
        "phfem_mesh_set_coefficients": [P, P, P, C.c_double],
        "phfem_mesh_connectivity": [P, P],
        "phfem_mesh_get_edges": [P, P, P],
        "phfem_mesh_get_faces": [P, P, P, P, P, P, P, P],
        "phfem_mesh_refinement_map": [P, P, P, P],
        "phfem_mesh_assemble": [P, C.c_int, P],
        "phfem_mesh_get_system": [P, P, P, P, P, P, P, P, P, P],
        "phfem_solve_ex": [P, C.c_int, C.c_double, I64, PP],
        "phfem_solution_stats": [P, P],
        "phfem_solution_errors_ex": [P, P],
        "phfem_pipeline": [P, C.c_int, C.c_int, P, P],
        "phfem_pipeline_child": [P, P, P, P, P, P],
        "phfem_solve_timed": [P, C.c_int, C.c_double, I64, P, P],
        "phfem_mesh_solve_faces": [P, C.c_int, C.c_double, I64, P, P],
        "phfem_mesh_solve_unverified": [P, C.c_int, C.c_double, I64, P, P, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.phfem_mesh_level.argtypes = [P]
    L.phfem_mesh_level.restype = C.c_int
    L.phfem_mesh_destroy.argtypes = [P]
    L.phfem_mesh_destroy.restype = None
    L.phfem_solution_destroy.argtypes = [P]
    L.phfem_solution_destroy.restype = None
    L.phfem_stream.restype = P
    _lib = L
    return L


# every symbol of include/phfem.h and include/phfem_ext.h
EXPORTED = [
    "phfem_last_error", "phfem_mesh_create_cube", "phfem_mesh_read", "phfem_mesh_write", "phfem_mesh_destroy",
    "phfem_mesh_refine", "phfem_mesh_level", "phfem_mesh_counts", "phfem_mesh_system_dims", "phfem_mesh_diameter",
    "phfem_mesh_dump_connectivity", "phfem_solve", "phfem_solution_destroy", "phfem_solution_values",
    "phfem_solution_stats_json", "phfem_solution_errors", "phfem_solution_write", "phfem_export_vtk",
    "phfem_export_multiplier_vtk", "phfem_dump_system",
    "phfem_mesh_create_from_arrays", "phfem_mesh_create_from_arrays_async", "phfem_mesh_create_kuhn", "phfem_mesh_sizes", "phfem_mesh_get_arrays",
    "phfem_mesh_set_coefficients", "phfem_mesh_connectivity", "phfem_mesh_get_edges", "phfem_mesh_get_faces",
    "phfem_mesh_refinement_map", "phfem_mesh_assemble", "phfem_mesh_get_system", "phfem_solve_ex",
    "phfem_solution_stats", "phfem_solution_errors_ex", "phfem_stream", "phfem_pipeline", "phfem_pipeline_child", "phfem_solve_timed",
    "phfem_mesh_solve_faces", "phfem_mesh_solve_unverified",
]


def _check(rc: int):
    if rc != OK:
        msg = lib().phfem_last_error().decode()
        raise _ERRORS.get(rc, PhfemError)(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def last_error() -> str:
    return lib().phfem_last_error().decode()


def stream_ptr() -> int:
    """cudaStream_t of the library (for CUDA-event timing on it)."""
    return lib().phfem_stream() or 0


# ---------------------------------------------------------------------------


class Mesh:
    """phfem_mesh handle (device resident)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.phfem_mesh_destroy(h)

    @property
    def handle(self):
        return self._h

    # constructors --------------------------------------------------------
    @classmethod
    def cube(cls) -> "Mesh":
        h = C.c_void_p()
        _check(lib().phfem_mesh_create_cube(C.byref(h)))
        return cls(h)

    @classmethod
    def read(cls, path: str) -> "Mesh":
        h = C.c_void_p()
        _check(lib().phfem_mesh_read(path.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays(cls, coords, tets, db, nb, level: int = 0) -> "Mesh":
        coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
        db = np.ascontiguousarray(db, dtype=np.int32).reshape(-1, 3)
        nb = np.ascontiguousarray(nb, dtype=np.int32).reshape(-1, 3)
        h = C.c_void_p()
        _check(lib().phfem_mesh_create_from_arrays(_ptr(coords), len(coords), _ptr(tets), len(tets), _ptr(db),
                                                   len(db), _ptr(nb), len(nb), level, C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays_async(cls, coords, tets, db, nb, level: int = 0) -> "Mesh":
        """Upload on the copy engine while the device keeps working; the
        arrays (page-locked for overlap) are kept alive by the returned mesh
        and must not change until its first use."""
        coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        tets = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
        db = np.ascontiguousarray(db, dtype=np.int32).reshape(-1, 3)
        nb = np.ascontiguousarray(nb, dtype=np.int32).reshape(-1, 3)
        h = C.c_void_p()
        _check(lib().phfem_mesh_create_from_arrays_async(_ptr(coords), len(coords), _ptr(tets), len(tets), _ptr(db),
                                                         len(db), _ptr(nb), len(nb), level, C.byref(h)))
        m = cls(h)
        m._host_arrays = (coords, tets, db, nb)
        return m

    @classmethod
    def kuhn(cls, nx, ny, nz, lx=1.0, ly=1.0, lz=1.0, jitter=0.0, seed=2509, dirichlet_mask=0x3F) -> "Mesh":
        h = C.c_void_p()
        _check(lib().phfem_mesh_create_kuhn(nx, ny, nz, lx, ly, lz, jitter, seed, dirichlet_mask, C.byref(h)))
        return cls(h)

    # reference API --------------------------------------------------------
    def write(self, path: str):
        _check(lib().phfem_mesh_write(self._h, path.encode()))

    def refine(self) -> RefineTimes:
        t = RefineTimes()
        _check(lib().phfem_mesh_refine(self._h, C.byref(t)))
        return t

    @property
    def level(self) -> int:
        return lib().phfem_mesh_level(self._h)

    def counts(self, with_connectivity=True):
        ne, nc, ned, nf = (C.c_int64() for _ in range(4))
        t = RefineTimes()
        if with_connectivity:
            _check(lib().phfem_mesh_counts(self._h, C.byref(ne), C.byref(nc), C.byref(ned), C.byref(nf), C.byref(t)))
            return dict(n_elems=ne.value, n_nodes=nc.value, n_edges=ned.value, n_faces=nf.value, times=t)
        _check(lib().phfem_mesh_counts(self._h, C.byref(ne), C.byref(nc), None, None, None))
        return dict(n_elems=ne.value, n_nodes=nc.value)

    def system_dims(self):
        n, l = C.c_int64(), C.c_int64()
        _check(lib().phfem_mesh_system_dims(self._h, C.byref(n), C.byref(l)))
        return n.value, l.value

    def diameter(self) -> float:
        h = C.c_double()
        _check(lib().phfem_mesh_diameter(self._h, C.byref(h)))
        return h.value

    def dump_connectivity(self, edges_csv=None, faces_csv=None):
        _check(lib().phfem_mesh_dump_connectivity(self._h, edges_csv.encode() if edges_csv else None,
                                                  faces_csv.encode() if faces_csv else None))

    def solve(self, problem=PROBLEM_MANUFACTURED, solver="schur", workers=1, tol=0.0) -> "Solution":
        h = C.c_void_p()
        _check(lib().phfem_solve(self._h, problem, solver.encode(), workers, tol, C.byref(h)))
        return Solution(h, self)

    def export_vtk(self, path, sol=None, with_point_data=False):
        _check(lib().phfem_export_vtk(self._h, sol.handle if sol else None, path.encode(), int(with_point_data)))

    def dump_system(self, problem, directory):
        _check(lib().phfem_dump_system(self._h, problem, directory.encode()))

    # extension API --------------------------------------------------------
    def sizes(self):
        s = np.zeros(4, dtype=np.int64)
        _check(lib().phfem_mesh_sizes(self._h, _ptr(s)))
        return tuple(int(v) for v in s)

    def arrays(self):
        nc, ne, nd, nn = self.sizes()
        coords = np.zeros((nc, 3))
        tets = np.zeros((ne, 4), dtype=np.int32)
        db = np.zeros((nd, 3), dtype=np.int32)
        nb = np.zeros((nn, 3), dtype=np.int32)
        _check(lib().phfem_mesh_get_arrays(self._h, _ptr(coords), _ptr(tets), _ptr(db), _ptr(nb)))
        return coords, tets, db, nb

    def set_coefficients(self, a_elem=None, a_diag=None, c=1.0):
        a_elem = None if a_elem is None else np.ascontiguousarray(a_elem, dtype=np.float64)
        a_diag = None if a_diag is None else np.ascontiguousarray(a_diag, dtype=np.float64)
        _check(lib().phfem_mesh_set_coefficients(self._h, _ptr(a_elem), _ptr(a_diag), c))

    def connectivity(self):
        c = np.zeros(6, dtype=np.int64)
        _check(lib().phfem_mesh_connectivity(self._h, _ptr(c)))
        return dict(ned=int(c[0]), nf=int(c[1]), n_interior=int(c[2]), n_dirichlet=int(c[3]),
                    n_neumann=int(c[4]), l=int(c[5]))

    def edges(self):
        ne = self.sizes()[1]
        ned = self.connectivity()["ned"]
        en = np.zeros((ned, 2), dtype=np.int32)
        eos = np.zeros((ne, 6), dtype=np.int32)
        _check(lib().phfem_mesh_get_edges(self._h, _ptr(en), _ptr(eos)))
        return en, eos

    def faces(self) -> dict:
        ne = self.sizes()[1]
        c = self.connectivity()
        nf = c["nf"]
        out = dict(faces=np.zeros((nf, 3), dtype=np.int32), face_of_slot=np.zeros(4 * ne, dtype=np.int32),
                   sigma=np.zeros(4 * ne, dtype=np.int8), face_slots=np.zeros((nf, 2), dtype=np.int64),
                   face_class=np.zeros(nf, dtype=np.uint8), mrow=np.zeros(nf, dtype=np.int32),
                   area=np.zeros(nf))
        _check(lib().phfem_mesh_get_faces(self._h, _ptr(out["faces"]), _ptr(out["face_of_slot"]), _ptr(out["sigma"]),
                                          _ptr(out["face_slots"]), _ptr(out["face_class"]), _ptr(out["mrow"]),
                                          _ptr(out["area"])))
        out.update(c)
        out["nf"] = nf
        return out

    def refinement_map(self):
        s = np.zeros(2, dtype=np.int64)
        _check(lib().phfem_mesh_refinement_map(self._h, _ptr(s), None, None))
        mid = np.zeros(int(s[0]), dtype=np.int32)
        cen = np.zeros(int(s[1]), dtype=np.int32)
        _check(lib().phfem_mesh_refinement_map(self._h, None, _ptr(mid), _ptr(cen)))
        return mid, cen

    def assemble(self, problem=PROBLEM_MANUFACTURED) -> dict:
        s = np.zeros(3, dtype=np.int64)
        _check(lib().phfem_mesh_assemble(self._h, problem, _ptr(s)))
        n, l, nnz = (int(v) for v in s)
        ne = n // 4
        out = dict(a_blocks=np.zeros((ne, 4, 4)), slot_coef=np.zeros((ne, 4)),
                   slot_mrow=np.zeros((ne, 4), dtype=np.int32), rhs=np.zeros(n), bd=np.zeros(l),
                   s_rowptr=np.zeros(l + 1, dtype=np.int64), s_col=np.zeros(nnz, dtype=np.int32),
                   s_val=np.zeros(nnz), rhs_neg=np.zeros(l))
        _check(lib().phfem_mesh_get_system(self._h, *(_ptr(out[k]) for k in (
            "a_blocks", "slot_coef", "slot_mrow", "rhs", "bd", "s_rowptr", "s_col", "s_val", "rhs_neg"))))
        return out

    def solve_ex(self, problem, tol=1e-10, max_iter=-1) -> "Solution":
        h = C.c_void_p()
        _check(lib().phfem_solve_ex(self._h, problem, tol, max_iter, C.byref(h)))
        return Solution(h, self)

    def solve_faces(self, problem, tol=1e-10, max_iter=-1):
        """Face system only (pcg_jacobi with inner_cg_options); no verify."""
        l = self.connectivity()["l"]
        lam = np.zeros(l)
        out = np.zeros(3)
        _check(lib().phfem_mesh_solve_faces(self._h, problem, tol, max_iter, _ptr(lam), _ptr(out)))
        return lam, dict(iterations=int(out[0]), rel_residual=out[1], converged=bool(out[2]))

    def pipeline(self, problem, do_refine=True, assemble=True):
        ms = StageMs()
        counts = np.zeros(5, dtype=np.int64)
        flags = (1 if do_refine else 0) | (0 if assemble else 2)
        _check(lib().phfem_pipeline(self._h, problem, flags, C.byref(ms), _ptr(counts)))
        return {n: getattr(ms, n) for n, _ in StageMs._fields_}, counts

    def pipeline_child(self):
        """The last pipeline pass's refined child (coords, tets, db, nb)."""
        sz = np.zeros(4, dtype=np.int64)
        _check(lib().phfem_pipeline_child(self._h, _ptr(sz), None, None, None, None))
        nc, ne, nd, nn = (int(v) for v in sz)
        c = np.zeros((nc, 3))
        t = np.zeros((ne, 4), dtype=np.int32)
        d = np.zeros((nd, 3), dtype=np.int32)
        n = np.zeros((nn, 3), dtype=np.int32)
        _check(lib().phfem_pipeline_child(self._h, _ptr(sz), _ptr(c), _ptr(t), _ptr(d), _ptr(n)))
        return c, t, d, n

    def solve_timed(self, problem, tol=1e-10, max_iter=-1):
        """Schur solve with timings: CG on the device, then recovery + verify
        (a verify refusal is reported as accepted=False, not raised)."""
        out = np.zeros(8)
        vt = np.zeros(4)
        _check(lib().phfem_solve_timed(self._h, problem, tol, max_iter, _ptr(out), _ptr(vt)))
        return dict(iterations=int(out[0]), cg_ms=out[1], ms_per_iteration=out[2], converged=bool(out[3]),
                    total_s=out[4], accepted=bool(out[5]), residual=out[6], constraint_residual=out[7],
                    r1=vt[0], r2=vt[1], norm_rhs=vt[2], norm_bd=vt[3])

    def solve_unverified(self, problem, tol=1e-10, max_iter=-1):
        """The whole Schur path (face solve + recovery + verify terms + error
        norms) without raising on verify_solution's refusal; returns U,
        Lambda and the stats."""
        n = 4 * self.sizes()[1]
        l = self.connectivity()["l"]
        u = np.zeros(n)
        lam = np.zeros(l)
        out = np.zeros(13)
        _check(lib().phfem_mesh_solve_unverified(self._h, problem, tol, max_iter, _ptr(u), _ptr(lam), _ptr(out)))
        keys = ("iterations", "residual", "constraint_residual", "converged", "accepted", "r1", "r2", "norm_rhs",
                "norm_bd", "cg_rel_residual", "err_y", "err_kappa", "err_l2")
        st = dict(zip(keys, (float(v) for v in out)))
        st["iterations"] = int(st["iterations"])
        st["converged"] = bool(st["converged"])
        st["accepted"] = bool(st["accepted"])
        return u, lam, st


class Solution:
    """phfem_solution handle; keeps its mesh's device snapshot alive."""

    def __init__(self, handle, mesh: Mesh):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.phfem_solution_destroy(h)

    @property
    def handle(self):
        return self._h

    def values(self):
        u, lam = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        n, l = C.c_int64(), C.c_int64()
        _check(lib().phfem_solution_values(self._h, C.byref(u), C.byref(n), C.byref(lam), C.byref(l)))
        U = np.ctypeslib.as_array(u, shape=(n.value,)).copy() if n.value else np.zeros(0)
        Lm = np.ctypeslib.as_array(lam, shape=(l.value,)).copy() if l.value else np.zeros(0)
        return U, Lm

    def stats_json(self) -> str:
        s = C.c_char_p()
        _check(lib().phfem_solution_stats_json(self._h, C.byref(s)))
        return s.value.decode()

    def stats(self):
        out = np.zeros(4)
        _check(lib().phfem_solution_stats(self._h, _ptr(out)))
        return dict(iterations=int(out[0]), residual=out[1], constraint_residual=out[2], seconds=out[3])

    def errors(self):
        eu, ek = C.c_double(), C.c_double()
        _check(lib().phfem_solution_errors(self._h, C.byref(eu), C.byref(ek)))
        return eu.value, ek.value

    def errors_ex(self):
        out = np.zeros(3)
        _check(lib().phfem_solution_errors_ex(self._h, _ptr(out)))
        return tuple(float(v) for v in out)

    def write(self, u_path=None, lambda_path=None):
        _check(lib().phfem_solution_write(self._h, u_path.encode() if u_path else None,
                                          lambda_path.encode() if lambda_path else None))

    def export_multiplier_vtk(self, path):
        _check(lib().phfem_export_multiplier_vtk(self._h, path.encode()))
