"""Output formats byte for byte against the reference's own writers (SURVEY
8(f) row 4): the same C-ABI calls on the same input go to this library and
to the unmodified reference library compiled into oracle/_ref (its capi.cpp,
vtk.cpp, mesh.cpp and sparse.cpp writers), and the files are compared.

* mesh text (phfem_mesh_write, mesh.cpp:117-130), connectivity CSVs
  (phfem_mesh_dump_connectivity, connectivity.cpp:211-225), the system dump
  (phfem_dump_system: COO of A and C, rhs, b_D; capi.cpp:280-308) and the
  VTK of the mesh alone (vtk.cpp:27-35): byte-identical;
* files carrying the solution (VTK cell / point data, multiplier VTK,
  phfem_solution_write): identical apart from the numbers, which agree to
  1e-9 relative in the l2 norm over the file (the solution bar; the solves
  are not bit for bit: the CG dot products are summed in another order).
Levels 0-2 of the reference's 5-tet cube, problem 0 (manufactured)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle_bind import REF_SO, ref_available

pytestmark = pytest.mark.gpu

ph = pytest.importorskip("paper_2509_11133_b200.phfem")

NUM = re.compile(r"[-+]?(?:\d+\.\d*|\.\d+|\d+)(?:[eE][-+]?\d+)?")


class _Ref:
    """the reference's C ABI (phfem.h) from oracle/_ref/libphfem_ref.so"""

    def __init__(self):
        L = C.CDLL(REF_SO)
        P, PP = C.c_void_p, C.POINTER(C.c_void_p)
        for name, args in {"phfem_mesh_create_cube": [PP], "phfem_mesh_refine": [P, P],
                           "phfem_mesh_write": [P, C.c_char_p],
                           "phfem_mesh_dump_connectivity": [P, C.c_char_p, C.c_char_p],
                           "phfem_solve": [P, C.c_int, C.c_char_p, C.c_int, C.c_double, PP],
                           "phfem_solution_write": [P, C.c_char_p, C.c_char_p],
                           "phfem_export_vtk": [P, P, C.c_char_p, C.c_int], "phfem_export_multiplier_vtk": [P, C.c_char_p],
                           "phfem_dump_system": [P, C.c_int, C.c_char_p]}.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int
        L.phfem_last_error.restype = C.c_char_p
        self.L = L

    def ok(self, rc):
        assert rc == 0, self.L.phfem_last_error().decode()


def _read(p):
    with open(p, "rb") as f:
        return f.read()


def _same_up_to_numbers(a: bytes, b: bytes, rtol=1e-9):
    """same lines apart from the numbers; the numbers of the file agree to
    rtol in the l2 norm (the solution bar: the solves agree to 1e-9, not per
    entry on entries near zero)"""
    la, lb = a.decode().splitlines(), b.decode().splitlines()
    assert len(la) == len(lb)
    xa, xb = [], []
    for x, y in zip(la, lb):
        assert NUM.sub("#", x) == NUM.sub("#", y), (x, y)
        xa += [float(u) for u in NUM.findall(x)]
        xb += [float(v) for v in NUM.findall(y)]
    xa, xb = np.array(xa), np.array(xb)
    rel = float(np.linalg.norm(xa - xb) / max(np.linalg.norm(xb), 1e-300))
    assert rel <= rtol, rel
    return rel


@pytest.mark.parametrize("level", [0, 1, 2])
def test_writers_match_reference(tmp_path, level):
    if not ref_available():
        pytest.skip("oracle/_ref/libphfem_ref.so not built")
    R = _Ref()
    rm = C.c_void_p()
    R.ok(R.L.phfem_mesh_create_cube(C.byref(rm)))
    g = ph.Mesh.cube()
    for _ in range(level):
        R.ok(R.L.phfem_mesh_refine(rm, None))
        g.refine()
    dirs = {}
    for who in ("ref", "ours"):
        d = tmp_path / who
        d.mkdir()
        (d / "sys").mkdir()
        dirs[who] = d
    r, o = dirs["ref"], dirs["ours"]
    R.ok(R.L.phfem_mesh_write(rm, str(r / "mesh.txt").encode()))
    g.write(str(o / "mesh.txt"))
    R.ok(R.L.phfem_mesh_dump_connectivity(rm, str(r / "edges.csv").encode(), str(r / "faces.csv").encode()))
    g.dump_connectivity(str(o / "edges.csv"), str(o / "faces.csv"))
    R.ok(R.L.phfem_dump_system(rm, 0, str(r / "sys").encode()))
    g.dump_system(0, str(o / "sys"))
    R.ok(R.L.phfem_export_vtk(rm, None, str(r / "mesh.vtk").encode(), 0))
    g.export_vtk(str(o / "mesh.vtk"))
    for name in ("mesh.txt", "edges.csv", "faces.csv", "sys/a.txt", "sys/c.txt", "sys/rhs.txt", "sys/bd.txt",
                 "mesh.vtk"):
        assert _read(r / name) == _read(o / name), name
    # solution-carrying files
    rs = C.c_void_p()
    R.ok(R.L.phfem_solve(rm, 0, b"schur", 1, 0.0, C.byref(rs)))
    sol = g.solve(ph.PROBLEM_MANUFACTURED, "schur", 1, 0.0)
    R.ok(R.L.phfem_export_vtk(rm, rs, str(r / "sol.vtk").encode(), 1))
    g.export_vtk(str(o / "sol.vtk"), sol, True)
    R.ok(R.L.phfem_export_multiplier_vtk(rs, str(r / "lam.vtk").encode()))
    sol.export_multiplier_vtk(str(o / "lam.vtk"))
    R.ok(R.L.phfem_solution_write(rs, str(r / "u.txt").encode(), str(r / "l.txt").encode()))
    sol.write(str(o / "u.txt"), str(o / "l.txt"))
    for name in ("sol.vtk", "lam.vtk", "u.txt", "l.txt"):
        _same_up_to_numbers(_read(r / name), _read(o / name))
