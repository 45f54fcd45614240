"""Host setup is bit-exact with the reference: basis tables, mesh side tables,
orientation flips, curl-form metrics, SFC partition, Domain lowering. CPU only."""

import numpy as np
import pytest

from conftest import golden
from paper_2404_12703_b200 import mesh as mm
from paper_2404_12703_b200.basis import build_basis
from paper_2404_12703_b200.equations import GasProperties
from paper_2404_12703_b200.operator import Domain

MESH_KEYS = ("side_elem_p", "side_loc_p", "side_elem_r", "side_loc_r", "side_orient", "side_bc",
             "elem_sides", "elem_primary", "grid_index")
DOMAIN_KEYS = ("side_global", "ef_side", "ef_sign", "ef_orient", "rows_inner", "rows_mpi",
               "sides_inner", "sides_mpi_primary", "sides_mpi_replica", "sides_bc", "side_bc")
BASIS_KEYS = ("nodes", "weights", "D", "Dhat", "Dsplit", "l_minus", "l_plus", "lhat_minus",
              "lhat_plus", "vandermonde_modal", "geom_to_solution")


def test_basis_bitwise():
    z = golden("basis")
    for N in range(1, 9):
        for nt in ("GL", "LGL"):
            b = build_basis(N, nt)
            for f in BASIS_KEYS:
                assert np.array_equal(getattr(b, f), z[f"{nt}{N}_{f}"]), (N, nt, f)


@pytest.mark.parametrize("case", ["orient3", "walls432", "randflip4"])
def test_mesh_tables_metrics_partition_domain(case):
    z = golden("tables_" + case)
    m = mm.generate_box_mesh(*[int(n) for n in z["spec_n"]], z["spec_ext"],
                             tuple(bool(p) for p in z["spec_per"]))
    m = mm.permute_elements(m, z["flip_elems"], [str(k) for k in z["flip_kinds"]])
    for k in MESH_KEYS:
        assert np.array_equal(getattr(m, k), z[k]), k
    mc = mm.curve_mesh(m, 0.05)
    mm.compute_metrics(mc, build_basis(3, "LGL"), backend="numpy")
    for k in ("J", "Ja", "x", "face_normal", "face_s"):
        assert np.array_equal(getattr(mc, k), z[k]), k
    parts = mm.partition_sfc(mc, 3)
    er = np.empty(mc.nelem, dtype=np.int64)
    for p in parts:
        er[p.lo:p.hi] = p.rank
    for p in parts:
        assert p.lo == z[f"part{p.rank}_lo"] and p.hi == z[f"part{p.rank}_hi"]
        assert sorted(p.neighbors) == sorted(
            int(k.split("nbr")[1]) for k in z if k.startswith(f"part{p.rank}_nbr"))
        for k, v in p.neighbors.items():
            assert np.array_equal(v, z[f"part{p.rank}_nbr{k}"])
        d = Domain(mc, build_basis(3, "LGL"), GasProperties(), p.lo, p.hi, er, p.rank)
        for k in DOMAIN_KEYS:
            assert np.array_equal(np.asarray(getattr(d, k)), z[f"dom{p.rank}_{k}"]), k
        for nb, info in d.neighbors.items():
            assert np.array_equal(info["sides"], z[f"dom{p.rank}_nbr{nb}_sides"])
            assert np.array_equal(info["is_primary"], z[f"dom{p.rank}_nbr{nb}_is_primary"])


def test_orientation_codes_all_present():
    m = mm.permute_element_axes(mm.generate_box_mesh(3, 3, 3, [(-1.0, 1.0)] * 3, (True,) * 3),
                                13, "flip_xy")
    assert set(np.unique(m.side_orient)) == {0, 1, 2, 3}


def test_random_flips_vectorised_matches_sequential():
    base = mm.generate_box_mesh(4, 4, 3, [(0.0, 1.0)] * 3, (True, False, True))
    rng = np.random.default_rng(3)
    seq = [(int(rng.integers(base.nelem)), ("flip_xy", "flip_xz", "flip_yz")[rng.integers(3)])
           for _ in range(30)]
    a = base
    for e, k in seq:
        a = mm.permute_element_axes(a, e, k)
    b = mm.permute_elements(base, [e for e, _ in seq], [k for _, k in seq])
    for k in MESH_KEYS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_c4_mesh_all_codes_and_positive_jacobian():
    m = mm.curve_mesh(mm.random_flips(mm.generate_box_mesh(6, 6, 6, [(0.0, 2 * np.pi)] * 3,
                                                           (True,) * 3)), 0.05)
    assert set(np.unique(m.side_orient)) == {0, 1, 2, 3}
    mm.compute_metrics(m, build_basis(4, "LGL"))
    assert np.all(m.J > 0.0)
    assert mm.metric_identity_residual(m) < 1e-12


def test_torch_metrics_agree_with_numpy():
    pytest.importorskip("torch")
    m = mm.curve_mesh(mm.generate_box_mesh(3, 2, 2, [(0.0, 1.0)] * 3, (True,) * 3), 0.08)
    a = mm.curve_mesh(m, 0.08)
    b = mm.curve_mesh(m, 0.08)
    mm.compute_metrics(a, build_basis(4, "LGL"), backend="numpy")
    mm.compute_metrics(b, build_basis(4, "LGL"), backend="torch")
    # different contraction order (BLAS / cuBLAS): roundoff-level agreement
    assert np.max(np.abs(a.Ja - b.Ja)) < 1e-12
    assert np.max(np.abs(a.J - b.J) / a.J) < 1e-12
    assert np.max(np.abs(a.face_normal - b.face_normal)) < 1e-12


def test_hdgm_cache_roundtrip(tmp_path):
    m = mm.curve_mesh(mm.generate_box_mesh(2, 2, 2, [(0.0, 1.0)] * 3, (True,) * 3), 0.05)
    b = build_basis(3, "LGL")
    mm.compute_metrics(m, b)
    p = tmp_path / "m.hdgm"
    mm.write_mesh_cache(m, b, p)
    m2 = mm.load_mesh_cache(p)
    mm.compute_metrics(m2, b)
    assert np.array_equal(m2.Ja, m.Ja)
    for k in ("side_elem_p", "side_loc_p", "side_elem_r", "side_orient", "elem_sides"):
        assert np.array_equal(getattr(m2, k), getattr(m, k))


def test_partition_uneven_counts():
    m = mm.generate_box_mesh(3, 3, 3, [(0.0, 1.0)] * 3, (True,) * 3)
    parts = mm.partition_sfc(m, 5)
    sizes = [p.n_elems for p in parts]
    assert sum(sizes) == 27 and max(sizes) - min(sizes) <= 1
    with pytest.raises(mm.MeshError):
        mm.partition_sfc(m, 28)
