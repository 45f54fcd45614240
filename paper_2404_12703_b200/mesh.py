"""Hexahedral box meshes, orientation flips, curl-form metrics, SFC partition.

Host-side setup that feeds the device tables. Same public API and the same
integer tables as ``hexdg.mesh`` (reference ``src/mesh.py``) -- the side
tables are checked bit-exact against the reference in ``tests/`` -- but every
routine is vectorised: the reference's per-element / per-side Python loops
(``generate_box_mesh`` :191-276, ``permute_element_axes`` :318-398, the
per-side face-metric loop :487-497, ``partition_sfc`` :518-551) dominate its
setup time (76 s at 32^3, hours for a 40^3 randomly flipped mesh).

Conventions (identical to the reference, src/mesh.py:10-22): locSides
0..5 = xi-, xi+, eta-, eta+, zeta-, zeta+; face coordinates (p, q) run along
the tangential axes (d+1)%3, (d+2)%3; orientation codes 0..3 = identity,
flip p, flip q, flip both.
"""

import copy
from dataclasses import dataclass, field

import numpy as np

from .basis import Basis1D, differentiation_matrix

N_LOC_SIDES = 6
ORIENTATION_CODES = (0, 1, 2, 3)
BC_NONE = 0


class MeshError(ValueError):
    pass


def morton_key(ix, iy, iz, nbits: int = 21):
    """Bit interleave with x least significant (src/mesh.py:42-49); vectorised."""
    ix, iy, iz = (np.asarray(a, dtype=np.int64) for a in (ix, iy, iz))
    key = np.zeros(np.broadcast(ix, iy, iz).shape, dtype=np.int64)
    for t in range(nbits):
        key |= ((ix >> t) & 1) << (3 * t)
        key |= ((iy >> t) & 1) << (3 * t + 1)
        key |= ((iz >> t) & 1) << (3 * t + 2)
    return key if key.shape else int(key)


def loc_side_axes(loc: int):
    d = loc // 2
    return d, loc % 2 == 1, (d + 1) % 3, (d + 2) % 3


def orient_map(code: int, p: int, q: int, N: int):
    if code == 0:
        return p, q
    if code == 1:
        return N - p, q
    if code == 2:
        return p, N - q
    if code == 3:
        return N - p, N - q
    raise MeshError(f"invalid orientation code {code}")


def side_mapping(loc_side: int, orientation: int, p: int, q: int, N: int):
    """Volume index line behind face node (p, q) (src/mesh.py:70-86)."""
    if not (0 <= p <= N and 0 <= q <= N):
        raise MeshError(f"face index ({p}, {q}) out of range for N={N}")
    a, b = orient_map(orientation, p, q, N)
    d, plus, t1, t2 = loc_side_axes(loc_side)
    line = np.empty((N + 1, 3), dtype=np.int64)
    line[:, d] = np.arange(N + 1)
    line[:, t1] = a
    line[:, t2] = b
    return line, d, plus


@dataclass
class Partition:
    rank: int
    lo: int
    hi: int
    neighbors: dict

    @property
    def n_elems(self) -> int:
        return self.hi - self.lo


@dataclass
class Mesh:
    """Field set of src/mesh.py:105-142."""

    nelem: int
    corners: np.ndarray
    extents: np.ndarray
    periodic: tuple
    counts: tuple
    grid_index: np.ndarray
    curve_amplitude: float

    n_sides: int
    side_elem_p: np.ndarray
    side_loc_p: np.ndarray
    side_elem_r: np.ndarray
    side_loc_r: np.ndarray
    side_orient: np.ndarray
    side_bc: np.ndarray
    side_shift: np.ndarray

    elem_sides: np.ndarray
    elem_primary: np.ndarray

    basis: Basis1D = field(default=None, repr=False)
    geom: np.ndarray = field(default=None, repr=False)
    x: np.ndarray = field(default=None, repr=False)
    J: np.ndarray = field(default=None, repr=False)
    Ja: np.ndarray = field(default=None, repr=False)
    face_normal: np.ndarray = field(default=None, repr=False)
    face_s: np.ndarray = field(default=None, repr=False)

    @property
    def n_interior_sides(self) -> int:
        return int(np.sum(self.side_elem_r >= 0))

    @property
    def n_boundary_sides(self) -> int:
        return int(np.sum(self.side_elem_r < 0))


def _deformation(points, amplitude, extents):
    """Sinusoidal bump vanishing on the walls (src/mesh.py:145-154)."""
    if amplitude == 0.0:
        return points
    lo = extents[:, 0]
    L = extents[:, 1] - extents[:, 0]
    u = (points - lo) / L
    bump = np.sin(2.0 * np.pi * u[..., 0]) * np.sin(2.0 * np.pi * u[..., 1]) \
        * np.sin(2.0 * np.pi * u[..., 2])
    return points + amplitude * bump[..., None] * L


# ---------------------------------------------------------------------------
# box generation


def generate_box_mesh(nx: int, ny: int, nz: int, extents, periodic) -> Mesh:
    """Morton-ordered Cartesian box (semantics of src/mesh.py:191-276).

    Side creation order is the reference's: per element in SFC order, per
    direction d: the +d side it owns as primary, then (non-periodic wall only)
    its -d boundary side.
    """
    counts = (int(nx), int(ny), int(nz))
    if min(counts) < 1:
        raise MeshError(f"element counts must be >= 1, got {counts}")
    extents = np.asarray(extents, dtype=np.float64).reshape(3, 2)
    if np.any(extents[:, 1] <= extents[:, 0]):
        raise MeshError("extents must be non-empty intervals")
    periodic = tuple(bool(p) for p in periodic)
    cnt = np.array(counts, dtype=np.int64)

    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    g = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)       # ix fastest
    order = np.argsort(morton_key(g[:, 0], g[:, 1], g[:, 2]), kind="stable")
    grid = np.ascontiguousarray(g[order])
    ne = grid.shape[0]
    elem_of = np.empty(counts[::-1], dtype=np.int64)                 # [iz, iy, ix]
    elem_of[grid[:, 2], grid[:, 1], grid[:, 0]] = np.arange(ne)

    edges = [np.linspace(extents[d, 0], extents[d, 1], counts[d] + 1) for d in range(3)]
    corners = np.empty((ne, 2, 2, 2, 3))
    for c2 in (0, 1):
        for c1 in (0, 1):
            for c0 in (0, 1):
                corners[:, c2, c1, c0, 0] = edges[0][grid[:, 0] + c0]
                corners[:, c2, c1, c0, 1] = edges[1][grid[:, 1] + c1]
                corners[:, c2, c1, c0, 2] = edges[2][grid[:, 2] + c2]

    L = extents[:, 1] - extents[:, 0]
    # per (element, direction): the +d side, then an optional -d wall side
    wall_minus = np.zeros((ne, 3), dtype=bool)
    for d in range(3):
        if not periodic[d]:
            wall_minus[:, d] = grid[:, d] == 0
    n_per = 1 + wall_minus.astype(np.int64)                          # (ne, 3)
    start = np.concatenate([[0], np.cumsum(n_per.ravel())[:-1]]).reshape(ne, 3)
    ns = int(n_per.sum())
    s_ep = np.empty(ns, np.int64)
    s_lp = np.empty(ns, np.int64)
    s_er = np.empty(ns, np.int64)
    s_lr = np.empty(ns, np.int64)
    s_bc = np.zeros(ns, np.int64)
    s_shift = np.zeros((ns, 3))
    earr = np.arange(ne)
    for d in range(3):
        plus = start[:, d]
        nbr = grid.copy()
        nbr[:, d] += 1
        at_wall = nbr[:, d] == cnt[d]
        s_ep[plus] = earr
        s_lp[plus] = 2 * d + 1
        if periodic[d]:
            nbr[at_wall, d] = 0
            s_shift[plus[at_wall], d] = L[d]
            s_er[plus] = elem_of[nbr[:, 2], nbr[:, 1], nbr[:, 0]]
            s_lr[plus] = 2 * d
        else:
            inner = ~at_wall
            s_er[plus[inner]] = elem_of[nbr[inner, 2], nbr[inner, 1], nbr[inner, 0]]
            s_lr[plus[inner]] = 2 * d
            s_er[plus[at_wall]] = -1
            s_lr[plus[at_wall]] = -1
            s_bc[plus[at_wall]] = 2 * d + 2
            wm = wall_minus[:, d]
            minus = plus[wm] + 1
            s_ep[minus] = earr[wm]
            s_lp[minus] = 2 * d
            s_er[minus] = -1
            s_lr[minus] = -1
            s_bc[minus] = 2 * d + 1

    mesh = Mesh(nelem=ne, corners=corners, extents=extents, periodic=periodic,
                counts=counts, grid_index=grid, curve_amplitude=0.0, n_sides=ns,
                side_elem_p=s_ep, side_loc_p=s_lp, side_elem_r=s_er, side_loc_r=s_lr,
                side_orient=np.zeros(ns, np.int64), side_bc=s_bc, side_shift=s_shift,
                elem_sides=None, elem_primary=None)
    _rebuild_elem_side_table(mesh)
    return mesh


def _rebuild_elem_side_table(mesh: Mesh):
    """ElemToSide from SideToElem with the reference's consistency errors (src/mesh.py:279-297)."""
    ne, ns = mesh.nelem, mesh.n_sides
    elem_sides = np.full((ne, N_LOC_SIDES), -1, dtype=np.int64)
    elem_primary = np.zeros((ne, N_LOC_SIDES), dtype=bool)
    sid = np.arange(ns, dtype=np.int64)
    has_r = mesh.side_elem_r >= 0
    slots = np.concatenate([mesh.side_elem_p * N_LOC_SIDES + mesh.side_loc_p,
                            mesh.side_elem_r[has_r] * N_LOC_SIDES + mesh.side_loc_r[has_r]])
    owners = np.concatenate([sid, sid[has_r]])
    uniq, first, cnt = np.unique(slots, return_index=True, return_counts=True)
    if np.any(cnt > 1):
        slot = int(uniq[np.argmax(cnt > 1)])
        raise MeshError(f"element {slot // 6} locSide {slot % 6} referenced by two sides")
    elem_sides.reshape(-1)[slots] = owners
    elem_primary.reshape(-1)[mesh.side_elem_p * N_LOC_SIDES + mesh.side_loc_p] = True
    if np.any(elem_sides < 0):
        bad = np.argwhere(elem_sides < 0)[0]
        raise MeshError(f"element {bad[0]} locSide {bad[1]} has no side")
    mesh.elem_sides = elem_sides
    mesh.elem_primary = elem_primary


def curve_mesh(mesh: Mesh, amplitude: float) -> Mesh:
    """Copy with a smooth interior deformation (src/mesh.py:300-315)."""
    if mesh.corners is None:
        raise MeshError("cannot curve a mesh loaded from a cache file")
    out = copy.copy(mesh)
    out.curve_amplitude = float(amplitude)
    out.basis = out.geom = out.x = out.J = out.Ja = None
    out.face_normal = out.face_s = None
    return out


# ---------------------------------------------------------------------------
# orientation-changing element relabelings

_FLIP_AXES = {"flip_xy": (1, 2), "flip_xz": (0, 2), "flip_yz": (0, 1)}  # axes of corners[e]


def _face_grids(corners_e: np.ndarray, loc: int) -> np.ndarray:
    """(..., 2, 2, 3) face corner grid [p, q] of local face ``loc`` (src/mesh.py:157-168)."""
    d, plus, t1, t2 = loc_side_axes(loc)
    out = np.empty(corners_e.shape[:-4] + (2, 2, 3))
    for cp in (0, 1):
        for cq in (0, 1):
            idx = [0, 0, 0]
            idx[d] = 1 if plus else 0
            idx[t1] = cp
            idx[t2] = cq
            out[..., cp, cq, :] = corners_e[..., idx[2], idx[1], idx[0], :]
    return out


def _orient_grid(grid: np.ndarray, code: int) -> np.ndarray:
    if code == 0:
        return grid
    if code == 1:
        return grid[..., ::-1, :, :]
    if code == 2:
        return grid[..., :, ::-1, :]
    return grid[..., ::-1, ::-1, :]


def _all_face_grids(corners: np.ndarray) -> np.ndarray:
    """(n, 6, 2, 2, 3) grids of every local face."""
    return np.stack([_face_grids(corners, loc) for loc in range(N_LOC_SIDES)], axis=1)


def _match_code(primary, replica, tol=1e-9):
    """First code c with |primary - orient(replica, c)| < tol (src/mesh.py:181-188); -1 if none."""
    code = np.full(primary.shape[:-3], -1, dtype=np.int64)
    for c in reversed(ORIENTATION_CODES):
        ok = np.max(np.abs(primary - _orient_grid(replica, c)), axis=(-3, -2, -1)) < tol
        code = np.where(ok, c, code)
    return code


def permute_elements(mesh: Mesh, elems, kinds) -> Mesh:
    """Apply a sequence of double-axis flips, re-deriving sides geometrically.

    Equivalent to folding :func:`permute_element_axes` over ``zip(elems, kinds)``
    (the final locSides/orientations depend only on the final corner
    geometry: each physical face coincides with exactly one local face of each
    element), but vectorised over all affected sides.
    """
    elems = np.asarray(elems, dtype=np.int64).reshape(-1)
    kinds = list(kinds)
    if len(kinds) != elems.size:
        raise MeshError("elems and kinds differ in length")
    if mesh.corners is None:
        raise MeshError("cannot permute a mesh loaded from a cache file")
    if mesh.side_shift is None:
        raise MeshError("mesh lacks periodic shift data")
    for k in kinds:
        if k not in _FLIP_AXES:
            raise MeshError(f"unknown permutation kind {k!r}")
    if elems.size == 0:
        return mesh
    touched = np.unique(elems)
    sides = mesh.elem_sides[touched]
    selfpair = mesh.side_elem_p[sides] == mesh.side_elem_r[sides]
    if np.any(selfpair):
        raise MeshError(f"element {int(touched[np.argmax(selfpair.any(axis=1))])} "
                        "pairs with itself; cannot permute")

    out = copy.copy(mesh)
    out.corners = mesh.corners.copy()
    out.side_loc_p = mesh.side_loc_p.copy()
    out.side_loc_r = mesh.side_loc_r.copy()
    out.side_orient = mesh.side_orient.copy()
    out.basis = out.geom = out.x = out.J = out.Ja = None
    out.face_normal = out.face_s = None
    # flips of one element compose; apply them in sequence order
    for e, k in zip(elems, kinds):
        out.corners[e] = np.flip(out.corners[e], axis=_FLIP_AXES[k])

    aff = np.unique(mesh.elem_sides[touched].reshape(-1))
    ep, er = mesh.side_elem_p[aff], mesh.side_elem_r[aff]
    # each side's physical face = its old primary / replica face grid
    old_p = _vec_face(mesh.corners, ep, mesh.side_loc_p[aff])
    new_p_all = _all_face_grids(out.corners[ep])                       # (n, 6, 2,2,3)
    loc_p = _find_loc(new_p_all, old_p, aff, "primary")
    out.side_loc_p[aff] = loc_p
    inner = er >= 0
    if np.any(inner):
        ai = aff[inner]
        old_r = _vec_face(mesh.corners, er[inner], mesh.side_loc_r[ai])
        new_r_all = _all_face_grids(out.corners[er[inner]])
        loc_r = _find_loc(new_r_all, old_r, ai, "replica")
        out.side_loc_r[ai] = loc_r
        prim = new_p_all[np.flatnonzero(inner), loc_p[inner]]
        repl = new_r_all[np.arange(ai.size), loc_r] + mesh.side_shift[ai][:, None, None, :]
        code = _match_code(prim, repl)
        if np.any(code < 0):
            bad = ai[np.argmax(code < 0)]
            raise MeshError(f"no supported orientation for side {int(bad)}")
        out.side_orient[ai] = code
    _rebuild_elem_side_table(out)
    return out


def _vec_face(corners, elems, locs):
    out = np.empty((elems.size, 2, 2, 3))
    for loc in range(N_LOC_SIDES):
        m = locs == loc
        if np.any(m):
            out[m] = _face_grids(corners[elems[m]], loc)
    return out


def _find_loc(cand, target, sides, role):
    """Index of the candidate face whose corner set equals the target face (any code)."""
    n = target.shape[0]
    loc = np.full(n, -1, dtype=np.int64)
    for L in reversed(range(N_LOC_SIDES)):
        ok = _match_code(cand[:, L], target) >= 0
        loc = np.where(ok, L, loc)
    if np.any(loc < 0):
        raise MeshError(f"lost {role} face of side {int(sides[np.argmax(loc < 0)])}")
    return loc


def permute_element_axes(mesh: Mesh, e: int, kind: str) -> Mesh:
    """Reverse two reference axes of element ``e`` (API of src/mesh.py:318-398)."""
    if mesh.corners is None:
        raise MeshError("cannot permute a mesh loaded from a cache file")
    if kind not in _FLIP_AXES:
        raise MeshError(f"unknown permutation kind {kind!r}")
    return permute_elements(mesh, [e], [kind])


def random_flips(mesh: Mesh, seed: int = 0, prob: float = 0.5) -> Mesh:
    """C4 recipe: each element flipped with probability ``prob``,
    kind uniform over flip_xy/flip_xz/flip_yz, ``np.random.default_rng(seed)``."""
    rng = np.random.default_rng(seed)
    pick = rng.random(mesh.nelem) < prob
    kind_ix = rng.integers(0, 3, mesh.nelem)
    names = ("flip_xy", "flip_xz", "flip_yz")
    elems = np.flatnonzero(pick)
    return permute_elements(mesh, elems, [names[k] for k in kind_ix[elems]])


# ---------------------------------------------------------------------------
# metrics


def _axis_derivative(Dg, A, axis, xp=np):
    """1-D operator along reference axis 0/1/2 of (e, k, j, i, ...) (src/mesh.py:401-407)."""
    if axis == 0:
        return xp.einsum("ia,ekja...->ekji...", Dg, A)
    if axis == 1:
        return xp.einsum("ja,ekai...->ekji...", Dg, A)
    return xp.einsum("ka,eaji...->ekji...", Dg, A)


def extract_face(Q, loc, lvec_minus, lvec_plus):
    """Per-element nodal field on one local face, indexed [q, p] (src/mesh.py:414-429)."""
    d, plus, _, _ = loc_side_axes(loc)
    lvec = lvec_plus if plus else lvec_minus
    if d == 0:
        return np.einsum("a,kja...->kj...", lvec, Q)
    if d == 1:
        return np.swapaxes(np.einsum("a,kai...->ki...", lvec, Q), 0, 1)
    return np.einsum("a,aji...->ji...", lvec, Q)


def _face_metric(Ja_d_faces, loc, basis):
    """Vectorised extract_face over a batch (s, k, j, i, 3) of primary Ja^d blocks."""
    d, plus, _, _ = loc_side_axes(loc)
    if basis.node_type == "LGL":
        n = basis.N if plus else 0        # l+- are exact unit vectors: exact slice
        if d == 0:
            return Ja_d_faces[:, :, :, n, :]
        if d == 1:
            return np.swapaxes(Ja_d_faces[:, :, n, :, :], 1, 2)
        return Ja_d_faces[:, n, :, :, :]
    if Ja_d_faces.shape[0] == 0:
        return np.empty((0,) + Ja_d_faces.shape[2:])
    return np.stack([extract_face(Ja_d_faces[s], loc, basis.l_minus, basis.l_plus)
                     for s in range(Ja_d_faces.shape[0])])


class _TorchNS:
    """numpy-like namespace over torch (fp64), for the large-mesh metric path."""

    def __init__(self, device):
        import torch
        self.t = torch
        self.device = device

    def einsum(self, spec, *ops):
        return self.t.einsum(spec, *ops)

    def stack(self, xs, axis):
        return self.t.stack(list(xs), dim=axis)

    def empty_like(self, a):
        return self.t.empty_like(a)

    def det(self, a):
        return self.t.linalg.det(a)

    def asarray(self, a):
        return self.t.as_tensor(np.ascontiguousarray(a), dtype=self.t.float64,
                                device=self.device)

    def host(self, a):
        return a.cpu().numpy()


class _NumpyNS:
    einsum = staticmethod(np.einsum)
    stack = staticmethod(lambda xs, axis: np.stack(xs, axis=axis))
    empty_like = staticmethod(np.empty_like)
    det = staticmethod(np.linalg.det)
    asarray = staticmethod(lambda a: a)
    host = staticmethod(lambda a: a)


def _element_metrics(X, basis, Dg, xp=_NumpyNS):
    """x, J, Ja on solver nodes for a block of elements (src/mesh.py:452-485)."""
    dX = xp.stack([_axis_derivative(Dg, X, a, xp) for a in range(3)], axis=1)
    Ja_g = xp.empty_like(dX)
    for n in range(3):
        m, l = (n + 1) % 3, (n + 2) % 3
        A = X[..., l][:, None, ...] * dX[..., m]
        Ja_g[:, 0, ..., n] = -(_axis_derivative(Dg, A[:, 2], 1, xp)
                              - _axis_derivative(Dg, A[:, 1], 2, xp))
        Ja_g[:, 1, ..., n] = -(_axis_derivative(Dg, A[:, 0], 2, xp)
                              - _axis_derivative(Dg, A[:, 2], 0, xp))
        Ja_g[:, 2, ..., n] = -(_axis_derivative(Dg, A[:, 1], 0, xp)
                              - _axis_derivative(Dg, A[:, 0], 1, xp))
    if basis.node_type == "LGL":
        # geometry nodes are the solution nodes: interpolation is the identity
        x_sol, dX_sol, Ja = X, dX, Ja_g
    else:
        T = xp.asarray(basis.geom_to_solution)

        def to_solver(A):
            for a in range(3):
                A = _axis_derivative(T, A, a, xp)
            return A
        x_sol = to_solver(X)
        dX_sol = xp.stack([to_solver(dX[:, a]) for a in range(3)], axis=1)
        Ja = xp.stack([to_solver(Ja_g[:, i]) for i in range(3)], axis=1)
    J = xp.det(xp.stack([dX_sol[:, a] for a in range(3)], axis=-2))
    return x_sol, J, Ja


# meshes with more nodes than this use the torch (BLAS / CUDA) metric path;
# below it the numpy path reproduces the reference's metrics bit for bit
BITWISE_METRICS_MAX_NODES = 1 << 21


def compute_metrics(mesh: Mesh, basis: Basis1D, chunk: int = None, backend: str = None):
    """Curl-form metrics + per-side normals (src/mesh.py:432-506), chunked over elements.

    backend "numpy" reproduces the reference bit for bit; "torch" (default
    above BITWISE_METRICS_MAX_NODES) evaluates the same contractions with
    torch on the GPU when present (agreement ~1e-15 relative).
    """
    n1 = basis.N + 1
    g = basis.geom_nodes
    ne = mesh.nelem
    if backend is None:
        backend = "numpy" if ne * n1 ** 3 <= BITWISE_METRICS_MAX_NODES else "torch"
    if backend == "torch":
        import torch
        xp = _TorchNS("cuda" if torch.cuda.is_available() else "cpu")
        chunk = chunk or max(1, (1 << 23) // n1 ** 3)
    else:
        xp = _NumpyNS
        chunk = chunk or 2048
    Dg = xp.asarray(differentiation_matrix(g))
    B = xp.asarray(np.stack([(1.0 - g) / 2.0, (1.0 + g) / 2.0], axis=1))
    if mesh.corners is None:
        if mesh.geom.shape[1] != n1:
            raise MeshError(
                f"cached mesh has degree {mesh.geom.shape[1] - 1}, basis has N={basis.N}")
    lgl = basis.node_type == "LGL"
    geom = mesh.geom if mesh.corners is None else np.empty((ne, n1, n1, n1, 3))
    x = geom if lgl else np.empty((ne, n1, n1, n1, 3))
    J = np.empty((ne, n1, n1, n1))
    Ja = np.empty((ne, 3, n1, n1, n1, 3))
    for lo in range(0, ne, chunk):
        hi = min(ne, lo + chunk)
        if mesh.corners is not None:
            X = xp.einsum("ka,jb,ic,eabc...->ekji...", B, B, B, xp.asarray(mesh.corners[lo:hi]))
            X = xp.host(X)
            geom[lo:hi] = _deformation(X, mesh.curve_amplitude, mesh.extents)
        xs, Js, Jas = _element_metrics(xp.asarray(geom[lo:hi]), basis, Dg, xp)
        if not lgl:
            x[lo:hi] = xp.host(xs)
        J[lo:hi] = xp.host(Js)
        Ja[lo:hi] = xp.host(Jas)
    if np.any(J <= 0.0):
        bad = int(np.argwhere(np.any(J.reshape(ne, -1) <= 0.0, axis=1))[0, 0])
        raise MeshError(f"mapping fold-over: J <= 0 in element {bad}")

    normal, s = _side_metrics(mesh, basis, Ja, np.arange(mesh.n_sides))
    mesh.basis = basis
    mesh.geom = geom
    mesh.x = x
    mesh.J = J
    mesh.Ja = Ja
    mesh.face_normal = normal
    mesh.face_s = s
    return J, Ja


def _side_metrics(mesh, basis, Ja, sides, elem_offset=0):
    """Unit normal and surface element from the primary element (src/mesh.py:487-497)."""
    n1 = basis.N + 1
    normal = np.empty((sides.size, n1, n1, 3))
    s = np.empty((sides.size, n1, n1))
    ep = mesh.side_elem_p[sides] - elem_offset
    lp = mesh.side_loc_p[sides]
    for loc in range(N_LOC_SIDES):
        m = np.flatnonzero(lp == loc)
        if m.size == 0:
            continue
        d, plus, _, _ = loc_side_axes(loc)
        Jad = _face_metric(Ja[ep[m], d], loc, basis)
        Ns = (1.0 if plus else -1.0) * Jad
        snorm = np.sqrt(np.sum(Ns * Ns, axis=-1))
        normal[m] = Ns / snorm[..., None]
        s[m] = snorm
    return normal, s


def metric_identity_residual(mesh: Mesh) -> float:
    if mesh.Ja is None:
        raise MeshError("compute_metrics must run first")
    D = mesh.basis.D
    res = sum(_axis_derivative(D, mesh.Ja[:, a], a) for a in range(3))
    return float(np.max(np.abs(res)))


# ---------------------------------------------------------------------------
# partitioning


def partition_bounds(nelem: int, n_ranks: int):
    base, rem = divmod(nelem, n_ranks)
    sizes = [base + (1 if r < rem else 0) for r in range(n_ranks)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def partition_sfc(mesh: Mesh, n_ranks: int):
    """Contiguous balanced SFC ranges + per-neighbour shared sides (src/mesh.py:518-551)."""
    if n_ranks < 1:
        raise MeshError(f"need at least one rank, got {n_ranks}")
    if n_ranks > mesh.nelem:
        raise MeshError(f"{n_ranks} ranks exceed {mesh.nelem} elements")
    bounds = partition_bounds(mesh.nelem, n_ranks)
    elem_rank = np.repeat(np.arange(n_ranks, dtype=np.int64), np.diff(bounds))
    er = mesh.side_elem_r
    inner = np.flatnonzero(er >= 0)
    rp = elem_rank[mesh.side_elem_p[inner]]
    rr = elem_rank[er[inner]]
    cut = rp != rr
    sides, rp, rr = inner[cut], rp[cut], rr[cut]
    parts = []
    for r in range(n_ranks):
        neighbors = {}
        mine_p = rp == r
        mine_r = rr == r
        other = np.where(mine_p, rr, rp)
        sel = mine_p | mine_r
        for k in np.unique(other[sel]):
            neighbors[int(k)] = np.sort(sides[sel & (other == k)]).astype(np.int64)
        parts.append(Partition(rank=r, lo=int(bounds[r]), hi=int(bounds[r + 1]),
                               neighbors=neighbors))
    return parts


# ---------------------------------------------------------------------------
# binary mesh cache ("HDGM", src/mesh.py:557-620)

_MAGIC = b"HDGM"
_FORMAT_VERSION = 1
_NODE_TYPE_IDS = {"LGL": 0, "GL": 1}


def write_mesh_cache(mesh: Mesh, basis: Basis1D, path):
    if mesh.geom is None:
        compute_metrics(mesh, basis)
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(np.array([_FORMAT_VERSION, basis.N, mesh.nelem, _NODE_TYPE_IDS["LGL"],
                           mesh.n_sides], dtype="<u4").tobytes())
        fh.write(mesh.geom.astype("<f8").tobytes())
        conn = np.stack([mesh.side_elem_p, mesh.side_loc_p, mesh.side_elem_r,
                         mesh.side_loc_r, mesh.side_orient, mesh.side_bc], axis=1)
        fh.write(conn.astype("<i4").tobytes())


def load_mesh_cache(path) -> Mesh:
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _MAGIC:
            raise MeshError(f"not a mesh cache file (magic {magic!r})")
        version, N, nelem, node_type, n_sides = np.frombuffer(fh.read(20), dtype="<u4")
        if version != _FORMAT_VERSION:
            raise MeshError(f"unsupported mesh cache version {version}")
        if node_type != _NODE_TYPE_IDS["LGL"]:
            raise MeshError(f"unsupported geometry node type id {node_type}")
        n1, ne, ns = int(N) + 1, int(nelem), int(n_sides)
        geom = np.frombuffer(fh.read(ne * n1 ** 3 * 3 * 8), dtype="<f8").reshape(
            ne, n1, n1, n1, 3).astype(np.float64)
        conn = np.frombuffer(fh.read(ns * 6 * 4), dtype="<i4").reshape(ns, 6).astype(np.int64)
    mesh = Mesh(nelem=ne, corners=None,
                extents=np.array([[np.min(geom[..., d]), np.max(geom[..., d])] for d in range(3)]),
                periodic=(False, False, False), counts=(0, 0, 0),
                grid_index=np.zeros((ne, 3), dtype=np.int64), curve_amplitude=0.0,
                n_sides=ns, side_elem_p=conn[:, 0].copy(), side_loc_p=conn[:, 1].copy(),
                side_elem_r=conn[:, 2].copy(), side_loc_r=conn[:, 3].copy(),
                side_orient=conn[:, 4].copy(), side_bc=conn[:, 5].copy(),
                side_shift=np.zeros((ns, 3)), elem_sides=None, elem_primary=None)
    mesh.geom = geom
    _rebuild_elem_side_table(mesh)
    return mesh
