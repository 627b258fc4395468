"""CPU-side checks of the drop-in boundary (no GPU): libphfem.so loads and
exports every function include/phfem.h, phfem_ext.h and phfem_gpu.h declare;
the reference's C ABI surface is covered name for name; the host-side config
logic (counter RNG, coefficient fields) matches the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2509_11133_b200", "lib", "libphfem.so")

REFERENCE_CABI = [  # /root/reference/proj/include/phfem.h:39-123
    "phfem_last_error", "phfem_mesh_create_cube", "phfem_mesh_read", "phfem_mesh_write", "phfem_mesh_destroy",
    "phfem_mesh_refine", "phfem_mesh_level", "phfem_mesh_counts", "phfem_mesh_system_dims", "phfem_mesh_diameter",
    "phfem_mesh_dump_connectivity", "phfem_solve", "phfem_solution_destroy", "phfem_solution_values",
    "phfem_solution_stats_json", "phfem_solution_errors", "phfem_solution_write", "phfem_export_vtk",
    "phfem_export_multiplier_vtk", "phfem_dump_system",
]


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(phfem_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(LIB):
        pytest.skip("libphfem.so not built")
    return ctypes.CDLL(LIB)


@pytest.mark.parametrize("header", ["phfem.h", "phfem_ext.h", "phfem_gpu.h"])
def test_every_declared_symbol_is_exported(so, header):
    names = declared(header)
    assert names
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_reference_c_abi_is_complete():
    names = declared("phfem.h")
    assert sorted(REFERENCE_CABI) == names


def test_python_binding_lists_all_symbols():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2509_11133_b200 import phfem as ph
    assert sorted(set(ph.EXPORTED)) == sorted(set(declared("phfem.h") + declared("phfem_ext.h")))


def test_counter_rng_matches_oracle(oracle):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2509_11133_b200 import configs
    idx = np.arange(1000)
    u = configs.uniform(11133, idx)
    assert np.array_equal(u, np.array([oracle.uniform(11133, int(i)) for i in idx]))
    a = configs.log_uniform_a(1000)
    assert a.min() >= 1e-2 and a.max() <= 1e2
    d = configs.aniso_diag(1000)
    assert set(map(tuple, d)) == {(1.0, 1.0, 100.0), (100.0, 1.0, 1.0)}
    assert 400 < (d[:, 2] == 100.0).sum() < 600


def test_config_table_sizes():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2509_11133_b200 import configs
    c4 = configs.CONFIGS[4]
    assert 6 * c4.nx * c4.ny * c4.nz == 12_582_912
    c3, c5 = configs.CONFIGS[3], configs.CONFIGS[5]
    assert 6 * c3.nx * c3.ny * c3.nz == 6 * c5.nx * c5.ny * c5.nz == 1_572_864
    assert 6 * 12 ** 7 == 214_990_848  # config 2, level 7
