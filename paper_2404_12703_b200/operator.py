"""Per-rank DG operator: connectivity lowering + device-resident state.

Mirror of ``hexdg.operator.Domain`` (reference ``src/operator.py:494-727``).

* The lowering (ElemToSide / SideToElem work lists, side classes, neighbour
  exchange order; reference :517-601) is vectorised numpy producing the same
  integer tables bit for bit, then packed into two int32 device tables
  (``ef_info``, ``side_info``, layout in include/hexdg_b200.h).
* Geometry, tables and workspaces live on the GPU (torch tensors used as
  plain device buffers); every kernel runs through the C ABI in
  ``csrc/libhexdg_b200.so``.
* The numpy attributes of the reference (``U, prim, Ut, UL, UR, fstar, g, gL,
  gR, vstar, bc_states`` ...) remain as host mirrors so the reference's tests
  and drivers run unchanged: API-level methods upload the inputs they read,
  launch, synchronise and download what they write. The production loop
  (``RankWorker.run`` / :meth:`Domain.stage`) never touches the mirrors.
"""

import ctypes

import numpy as np

from . import _lib
from . import equations as eq
from .basis import Basis1D, pack_basis
from .equations import N_LIFT
from .mesh import Mesh

NVAR = 5
NPRIM = 7

KIND_INNER, KIND_BC, KIND_MPI_PRIMARY, KIND_MPI_REPLICA = 0, 1, 2, 3

VOL_SURF, VOL_JAC, VOL_ACCUM, VOL_FVONLY = 1, 2, 4, 8


class OperatorError(RuntimeError):
    pass


def _orient(code, a, b, N):
    """Orientation map (src/operator.py:44-52); host helper for tests."""
    if code == 1:
        return N - a, b
    if code == 2:
        return a, N - b
    if code == 3:
        return N - a, N - b
    return a, b


def k_surf_int(fstar, ef_side, ef_sign, ef_orient, lhat_minus, lhat_plus, Ut):
    """Raw gather surface integral (reference ``k_surf_int``, src/operator.py:334-358):
    ``Ut += sum_loc ef_sign * lhat[m] * fstar[ef_side, q, p]`` on host arrays, one
    writer per DOF, evaluated by the device kernel behind ``hdg_surf_int`` (exact
    kernel set: the reference's operation order). ``Ut`` is updated in place."""
    from .basis import Basis1D  # noqa: F401  (layout documented by pack_basis)
    torch = _lib.require_cuda()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    Ut = np.asarray(Ut)
    ne, n1 = Ut.shape[0], Ut.shape[1]
    n2 = n1 * n1
    table = np.zeros(4 * n2 + 6 * n1)
    table[4 * n2 + 3 * n1:4 * n2 + 4 * n1] = lhat_minus
    table[4 * n2 + 4 * n1:4 * n2 + 5 * n1] = lhat_plus
    ef_info = ((np.asarray(ef_side, dtype=np.int64) << 3)
               | ((np.asarray(ef_sign) < 0).astype(np.int64) << 2)
               | np.asarray(ef_orient, dtype=np.int64)).astype(np.int32)
    keep = [torch.as_tensor(np.ascontiguousarray(a), device=dev)
            for a in (table, ef_info, np.asarray(fstar, dtype=np.float64),
                      np.ascontiguousarray(Ut, dtype=np.float64))]
    basis_d, ef_d, fs_d, ut_d = keep
    desc = _lib.HdgDomain()
    desc.N, desc.node_type, desc.ne, desc.ns = n1 - 1, 0, ne, int(np.asarray(fstar).shape[0])
    desc.basis, desc.ef_info = _lib.ptr(basis_d), _lib.ptr(ef_d)
    _lib.check(lib.hdg_surf_int(ctypes.byref(desc), _lib.ptr(fs_d), _lib.ptr(ut_d),
                                _lib.stream_ptr()), "hdg_surf_int")
    Ut[...] = ut_d.cpu().numpy()
    return Ut


class Domain:
    """Local element range, lowered tables, host mirrors and device state."""

    def __init__(self, mesh: Mesh, basis: Basis1D, gas: eq.GasProperties,
                 lo: int = 0, hi: int = None, elem_rank=None, rank: int = 0):
        if mesh.J is None:
            raise OperatorError("mesh metrics missing; call compute_metrics first")
        hi = mesh.nelem if hi is None else hi
        self.mesh, self.basis, self.gas = mesh, basis, gas
        self.rank = rank
        self.lo, self.hi = lo, hi
        self.ne = hi - lo
        n1 = basis.N + 1
        self.n1, self.N = n1, basis.N
        self._lower(mesh, lo, hi, elem_rank)

        self.J = np.ascontiguousarray(mesh.J[lo:hi])
        self.Ja = np.ascontiguousarray(mesh.Ja[lo:hi])
        self.x = np.ascontiguousarray(mesh.x[lo:hi])
        self.ssurf = np.ascontiguousarray(mesh.face_s[self.side_global])
        self.nvec = np.ascontiguousarray(mesh.face_normal[self.side_global])
        self.side_bc = np.ascontiguousarray(mesh.side_bc[self.side_global])

        ne, ns = self.ne, self.ns
        self.viscous = gas.viscous
        self.U = np.zeros((ne, n1, n1, n1, NVAR))
        self.prim = np.zeros((ne, n1, n1, n1, NPRIM))
        self.Ut = np.zeros((ne, n1, n1, n1, NVAR))
        self.UL = np.zeros((ns, n1, n1, NVAR))
        self.UR = np.zeros((ns, n1, n1, NVAR))
        self.fstar = np.zeros((ns, n1, n1, NVAR))
        nv = ne if self.viscous else 0
        nsv = ns if self.viscous else 0
        self.g = np.zeros((nv, n1, n1, n1, 3, N_LIFT))
        self.gL = np.zeros((nsv, n1, n1, 3, N_LIFT))
        self.gR = np.zeros((nsv, n1, n1, 3, N_LIFT))
        self.vstar = np.zeros((nsv, n1, n1, N_LIFT))
        self.Fvis = np.zeros((nv, n1, n1, n1, 3, NVAR))   # contravariant viscous fluxes
        self.bc_states = np.zeros((8, NVAR))
        self.exact = False          # kernel set for the API-level methods (see RankWorker)
        self._dev = None

    # ------------------------------------------------------------------
    # connectivity lowering (src/operator.py:517-601), vectorised

    def _lower(self, mesh, lo, hi, elem_rank):
        ep_all, er_all = mesh.side_elem_p, mesh.side_elem_r
        p_loc_all = (ep_all >= lo) & (ep_all < hi)
        r_loc_all = (er_all >= 0) & (er_all >= lo) & (er_all < hi)
        local = np.flatnonzero(p_loc_all | r_loc_all)
        self.side_global = local.astype(np.int64)
        self.ns = ns = local.size
        loc_of = np.full(mesh.n_sides, -1, dtype=np.int64)
        loc_of[local] = np.arange(ns)

        es = mesh.elem_sides[lo:hi]
        prim_side = mesh.elem_primary[lo:hi]
        self.ef_side = loc_of[es]
        self.ef_sign = np.where(prim_side, 1.0, -1.0)
        self.ef_orient = np.where(prim_side, 0, mesh.side_orient[es]).astype(np.int64)

        ep, er = ep_all[local], er_all[local]
        lp, lr, orr = mesh.side_loc_p[local], mesh.side_loc_r[local], mesh.side_orient[local]
        p_loc, r_loc = p_loc_all[local], r_loc_all[local]
        bc = er < 0
        inner2 = ~bc & p_loc & r_loc
        mpi = ~bc & ~inner2
        sl = np.arange(ns, dtype=np.int64)
        # rows_inner: per local side in order -- BC: primary row; interior: primary then replica
        n_rows = np.where(bc, 1, np.where(inner2, 2, 0))
        start = np.concatenate([[0], np.cumsum(n_rows)[:-1]])
        rows_inner = np.empty((int(n_rows.sum()), 5), dtype=np.int64)
        has = n_rows > 0
        pr_rows = start[has]
        rows_inner[pr_rows] = np.stack([sl[has], ep[has] - lo, lp[has],
                                        np.ones(has.sum(), np.int64),
                                        np.zeros(has.sum(), np.int64)], axis=1)
        rr_rows = start[inner2] + 1
        rows_inner[rr_rows] = np.stack([sl[inner2], er[inner2] - lo, lr[inner2],
                                        np.zeros(inner2.sum(), np.int64), orr[inner2]], axis=1)
        self.rows_inner = rows_inner
        mp = mpi & p_loc
        mr = mpi & ~p_loc
        rows_mpi = np.empty((int(mpi.sum()), 5), dtype=np.int64)
        ix = np.flatnonzero(mpi)
        rows_mpi[:, 0] = ix
        rows_mpi[:, 1] = np.where(mp[ix], ep[ix] - lo, er[ix] - lo)
        rows_mpi[:, 2] = np.where(mp[ix], lp[ix], lr[ix])
        rows_mpi[:, 3] = mp[ix].astype(np.int64)
        rows_mpi[:, 4] = np.where(mp[ix], 0, orr[ix])
        self.rows_mpi = rows_mpi
        self.side_is_mpi = mpi
        self.sides_inner = sl[bc | inner2]
        self.sides_mpi_primary = sl[mp]
        self.sides_mpi_replica = sl[mr]
        self.sides_mpi = sl[mpi]
        self.sides_bc = sl[bc]

        self.neighbors = {}
        if elem_rank is not None and mpi.any():
            other = np.where(mp, elem_rank[np.where(er >= 0, er, 0)],
                             elem_rank[ep])[mpi]
            gl, lcl, isp = local[mpi], sl[mpi], mp[mpi]
            for r in np.unique(other):
                m = other == r
                order = np.argsort(gl[m], kind="stable")
                self.neighbors[int(r)] = {"sides": lcl[m][order].astype(np.int64),
                                          "is_primary": isp[m][order].astype(bool)}

        # packed device tables
        kind = np.where(bc, KIND_BC, np.where(inner2, KIND_INNER,
                                              np.where(p_loc, KIND_MPI_PRIMARY, KIND_MPI_REPLICA)))
        bc_tag = mesh.side_bc[local]
        meta = (lp & 7) | ((np.where(lr >= 0, lr, 0) & 7) << 3) | ((orr & 3) << 6) \
            | ((bc_tag & 15) << 8) | (kind << 12)
        side_info = np.empty((ns, 4), dtype=np.int32)
        side_info[:, 0] = np.where(p_loc, ep - lo, -1)
        side_info[:, 1] = np.where(r_loc, er - lo, -1)
        side_info[:, 2] = meta
        side_info[:, 3] = -1
        self.side_info = side_info
        self.ef_info = ((self.ef_side << 3) | ((~prim_side).astype(np.int64) << 2)
                        | self.ef_orient).astype(np.int32)

    # ------------------------------------------------------------------
    # device state

    @property
    def device(self):
        if self._dev is None:
            self._dev = DeviceState(self)
        return self._dev

    def params(self, split=True, surf_solver=eq.RIEMANN_LLF, fv_solver=eq.RIEMANN_LLF,
               shock=None, source=None, exact=None, cfl=0.0, cfl_visc=0.0):
        """hdg_params for this domain's gas (shock: ShockConfig or None; source: (A, a) or None)."""
        g = self.gas
        p = _lib.HdgParams()
        p.gamma, p.R, p.Pr, p.mu_ref, p.T_ref = g.gamma, g.R, g.Pr, g.mu_ref, g.T_ref
        p.law = int(g.viscosity_law)
        p.viscous = int(self.viscous)
        p.split = int(split)
        p.surf_solver = int(surf_solver)
        p.fv_solver = int(fv_solver)
        if shock is not None and shock.enabled:
            from .shock import INDICATOR_CONSTANT, SHARPNESS, modal_threshold
            thr = modal_threshold(self.N)
            p.shock = 1
            p.indicator = 1 if shock.indicator == INDICATOR_CONSTANT else 0
            p.alpha_max, p.alpha_min = shock.alpha_max, shock.alpha_min
            p.alpha_const = shock.alpha_const
            p.ind_threshold = thr
            p.ind_slope = -SHARPNESS / thr
        if source is not None:
            p.source = 1
            p.mms_A, p.mms_a = source
        p.exact = int(self.exact if exact is None else exact)
        p.cfl, p.cfl_visc = float(cfl), float(cfl_visc)
        return p

    # ------------------------------------------------------------------
    # reference kernel wrappers (src/operator.py:629-727) -- API granularity,
    # host mirrors in/out, synchronous

    def _status(self):
        st = self.device.status.cpu().numpy()
        return st

    def cons_to_prim(self):
        dv = self.device
        dv.upload_state()
        torch = dv.torch
        prim = torch.empty((self.ne * self.n1 ** 3, NPRIM), dtype=torch.float64, device=dv.dev)
        _lib.check(dv.lib.hdg_cons_to_prim(dv.dptr, ctypes.byref(self.params()), _lib.ptr(dv.U),
                                           _lib.ptr(prim), dv.sptr()), "hdg_cons_to_prim")
        self.prim[...] = prim.cpu().numpy().reshape(self.prim.shape)
        self._raise_prim(self._status())

    def _raise_prim(self, st):
        if st[_lib.STATUS_BAD_PRIM]:
            ir = 1.0 / self.U[..., 0]
            p = (self.gas.gamma - 1.0) * (self.U[..., 4] - 0.5 * self.U[..., 0] * (
                (self.U[..., 1] * ir) ** 2 + (self.U[..., 2] * ir) ** 2 + (self.U[..., 3] * ir) ** 2))
            raise eq.AdmissibilityError(
                f"rank {self.rank}: inadmissible state (min rho {np.min(self.U[..., 0]):.3e}, "
                f"min p {np.min(p):.3e})")

    def prolong(self, mpi: bool):
        dv = self.device
        dv.upload_state()
        rows = dv.rows_mpi if mpi else dv.rows_inner
        n = self.rows_mpi.shape[0] if mpi else self.rows_inner.shape[0]
        if n:
            dv.upload_traces()
            _lib.check(dv.lib.hdg_prolong(dv.dptr, _lib.ptr(dv.U), _lib.ptr(rows), n, dv.sptr()),
                       "hdg_prolong")
        if not mpi:
            self._apply_bc_dev()
        if n or not mpi:
            self.UL[...] = dv.UL.cpu().numpy().reshape(self.UL.shape)
            self.UR[...] = dv.UR.cpu().numpy().reshape(self.UR.shape)

    def _apply_bc_dev(self):
        dv = self.device
        if self.sides_bc.size:
            dv.upload_bc()
            _lib.check(dv.lib.hdg_apply_bc_traces(dv.dptr, _lib.ptr(dv.sides_bc),
                                                  self.sides_bc.size, dv.sptr()),
                       "hdg_apply_bc_traces")

    def apply_bc_traces(self):
        for sl in self.sides_bc:
            self.UR[sl, :, :, :] = self.bc_states[self.side_bc[sl]]

    def fill_flux(self, sides, solver_id):
        sides = np.asarray(sides)
        if not sides.size:
            return
        dv = self.device
        dv.upload_traces(from_host=True)
        dv.upload_bc()
        dv.status.copy_(dv.status_init)
        sd = dv.int_tensor(sides)
        _lib.check(dv.lib.hdg_fill_flux_traces(dv.dptr, ctypes.byref(self.params()), _lib.ptr(sd),
                                               sides.size, int(solver_id), dv.sptr()),
                   "hdg_fill_flux_traces")
        self.fstar[...] = dv.fstar.cpu().numpy().reshape(self.fstar.shape)
        bad = int(self._status()[_lib.STATUS_BAD_SIDE])
        if bad >= 0:
            raise eq.AdmissibilityError(
                f"rank {self.rank}: inadmissible trace state on local side {bad}")

    def lift_gradients(self):
        """Full BR1 lifting (volume + surface + 1/J) and the nodal viscous fluxes."""
        if not self.viscous:
            return
        dv = self.device
        dv.upload_state()
        dv.upload_bc()
        dv.ensure_gradients()
        fn = dv.lib.hdg_phase_elem if self.basis.node_type == "LGL" else dv.lib.hdg_phase_lift
        _lib.check(fn(dv.dptr, ctypes.byref(self.params()), _lib.ptr(dv.U), dv.sptr()),
                   "lifting")
        dv.download_gradients()

    # the reference's split lifting calls (src/operator.py:667-685), on the host
    # mirrors, each through its own device kernel (api_kernels.cuh)
    def lift_fill(self, sides):
        """k_lift_fill: vstar on ``sides`` = mean of the (u, v, w, T) of UL and UR."""
        sides = np.asarray(sides)
        if not sides.size or not self.viscous:
            return
        dv = self.device
        dv.ensure_gradients()
        dv.upload_traces(from_host=True)
        dv.vstar.copy_(dv.torch.as_tensor(self.vstar))
        sd = dv.int_tensor(sides)
        _lib.check(dv.lib.hdg_lift_fill(dv.dptr, ctypes.byref(self.params()), _lib.ptr(sd),
                                        sides.size, dv.sptr()), "hdg_lift_fill")
        self.vstar[...] = dv.vstar.cpu().numpy()

    def lift_volume(self):
        """k_lift_volume: g = weak volume term of the lifting (no surface term, no 1/J)."""
        if not self.viscous:
            return
        dv = self.device
        dv.ensure_gradients()
        dv.upload_state()
        _lib.check(dv.lib.hdg_lift_volume(dv.dptr, ctypes.byref(self.params()), _lib.ptr(dv.U),
                                          dv.sptr()), "hdg_lift_volume")
        self.g[...] = dv.g.cpu().numpy()

    def lift_finish(self):
        """k_lift_surf_and_jac + k_viscous_contravariant: surface term from vstar, 1/J,
        and the nodal contravariant viscous fluxes Fvis."""
        if not self.viscous:
            return
        dv = self.device
        torch = dv.torch
        dv.ensure_gradients()
        dv.upload_state()
        dv.g.copy_(torch.as_tensor(self.g))
        dv.vstar.copy_(torch.as_tensor(self.vstar))
        fv = dv.Fvis if dv.Fvis is not None else torch.zeros(
            (self.ne, 3, 4, self.n1 ** 3), dtype=torch.float64, device=dv.dev)
        dv.desc.Fvis = _lib.ptr(fv)
        try:
            _lib.check(dv.lib.hdg_lift_finish(dv.dptr, ctypes.byref(self.params()),
                                              _lib.ptr(dv.U), dv.sptr()), "hdg_lift_finish")
        finally:
            dv._fill_desc()
        self.g[...] = dv.g.cpu().numpy()
        f = fv.cpu().numpy().reshape(self.ne, 3, 4, self.n1, self.n1, self.n1)
        self.Fvis[..., 0] = 0.0
        self.Fvis[..., 1:] = f.transpose(0, 3, 4, 5, 1, 2)

    def prolong_grad(self, mpi: bool):
        """Gradient traces; computed by the fused lifting kernel (see lift_gradients)."""
        if not mpi:
            self.lift_gradients()

    def vol_int(self, split: bool):
        """Ut += volume integral only (no surface term, no Jacobian)."""
        self._volume(self.params(split=split), VOL_ACCUM)

    def surf_int(self):
        dv = self.device
        ut = dv.torch.as_tensor(self.Ut, device=dv.dev).contiguous()
        fs = dv.torch.as_tensor(self.fstar, device=dv.dev).contiguous()
        _lib.check(dv.lib.hdg_surf_int(dv.dptr, _lib.ptr(fs), _lib.ptr(ut), dv.sptr()),
                   "hdg_surf_int")
        self.Ut[...] = ut.cpu().numpy()

    def apply_jac(self):
        dv = self.device
        ut = dv.torch.as_tensor(self.Ut, device=dv.dev).contiguous()
        _lib.check(dv.lib.hdg_apply_jac(dv.dptr, _lib.ptr(ut), dv.sptr()), "hdg_apply_jac")
        self.Ut[...] = ut.cpu().numpy()

    def _volume(self, prm, flags, t=0.0):
        dv = self.device
        dv.upload_state()
        ut = dv.torch.as_tensor(self.Ut, device=dv.dev).contiguous()
        _lib.check(dv.lib.hdg_phase_volume(dv.dptr, ctypes.byref(prm), _lib.ptr(dv.U), _lib.ptr(ut),
                                           None, t, 0.0, 0.0, 0.0, _lib.MODE_STORE_UT | (flags << 4),
                                           dv.sptr()), "hdg_phase_volume")
        self.Ut[...] = ut.cpu().numpy()

    def local_dt(self, cfl, cfl_visc):
        dv = self.device
        dv.upload_state()
        return dv.local_dt(dv.U, cfl, cfl_visc, self.params())


class DeviceState:
    """Device buffers of one Domain plus the packed hdg_domain descriptor."""

    def __init__(self, d: Domain):
        torch = _lib.require_cuda()
        self.torch = torch
        self.lib = _lib.load()
        self.d = d
        self.dev = torch.device("cuda", torch.cuda.current_device())
        f64 = dict(dtype=torch.float64, device=self.dev)
        n1, ne, ns = d.n1, d.ne, d.ns
        up = self.upload_array
        self.basis = up(pack_basis(d.basis))
        self.Ja = up(d.Ja)
        self.J = up(d.J)
        self.invJ = up(1.0 / d.J)
        self.nvec = up(d.nvec)
        self.ssurf = up(d.ssurf)
        self.x = up(d.x)
        self.ef_info = self.int_tensor(d.ef_info)
        self.side_info = self.int_tensor(d.side_info)
        self.bc = up(d.bc_states)
        self.rows_inner = self.int_tensor(d.rows_inner)
        self.rows_mpi = self.int_tensor(d.rows_mpi)
        self.sides_inner = self.int_tensor(d.sides_inner)
        self.sides_bc = self.int_tensor(d.sides_bc)
        self.sides_mpi_primary = self.int_tensor(d.sides_mpi_primary)
        self.U = torch.zeros((ne, n1, n1, n1, NVAR), **f64)
        self.UL = torch.zeros((ns, n1, n1, NVAR), **f64)
        self.UR = torch.zeros((ns, n1, n1, NVAR), **f64)
        self.fstar = torch.zeros((ns, n1, n1, NVAR), **f64)
        lgl = d.basis.node_type == "LGL"
        self.Fvis = self.fvface = self.vol = None
        if lgl:
            # element-pass output of the A -> flux -> C stage split (Euler and NS)
            self.vol = torch.zeros((ne, n1, n1, n1, NVAR), **f64)
        if d.viscous:
            self.fvface = torch.zeros((ns, 2, n1, n1, 4), **f64)
            if not lgl:
                self.Fvis = torch.zeros((ne, 3, 4, n1 ** 3), **f64)
        self.g = self.gL = self.gR = self.vstar = None
        self.alpha = torch.zeros(max(ne, 1), **f64)
        self.rfv = self.fv_list = self.fv_count = None   # allocated by set_fvm (shock)
        self.work = torch.zeros(4, dtype=torch.int32, device=self.dev)   # persistent-kernel counters
        self.fvm = None
        self.status_init = torch.tensor([0, -1, 0, 0, 0, 0, 0, 0], dtype=torch.int32, device=self.dev)
        self.status = self.status_init.clone()
        self.dt_bits = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.dt_valid = False   # host bookkeeping: dt_bits[0] = local dt of the current U
        self.desc = _lib.HdgDomain()
        self._fill_desc()

    # -- helpers --
    def upload_array(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.dev)

    def int_tensor(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=self.dev)

    def sptr(self):
        return _lib.stream_ptr()

    @property
    def dptr(self):
        return ctypes.byref(self.desc)

    def _fill_desc(self):
        d, D, P = self.d, self.desc, _lib.ptr
        D.N, D.node_type = d.N, 0 if d.basis.node_type == "LGL" else 1
        D.ne, D.ns = d.ne, d.ns
        D.basis, D.Ja, D.J, D.invJ = P(self.basis), P(self.Ja), P(self.J), P(self.invJ)
        D.nvec, D.ssurf, D.x = P(self.nvec), P(self.ssurf), P(self.x)
        D.ef_info, D.side_info, D.bc_states = P(self.ef_info), P(self.side_info), P(self.bc)
        D.UL, D.UR, D.fstar = P(self.UL), P(self.UR), P(self.fstar)
        D.Fvis, D.fvface = P(self.Fvis), P(self.fvface)
        D.g, D.gL, D.gR, D.vstar = P(self.g), P(self.gL), P(self.gR), P(self.vstar)
        D.alpha, D.status, D.dt_bits = P(self.alpha), P(self.status), P(self.dt_bits)
        D.vol = P(self.vol)
        D.rfv, D.fv_list, D.fv_count = P(self.rfv), P(self.fv_list), P(self.fv_count)
        D.work = P(self.work)
        if self.fvm is not None:
            D.fvm0, D.fvm1, D.fvm2 = (P(t) for t in self.fvm)

    def set_fvm(self, fvm):
        """Subcell metrics + the FV workspaces (residual, flagged-element list)."""
        self.fvm = tuple(self.upload_array(a) for a in fvm)
        if self.rfv is None:
            d, torch = self.d, self.torch
            self.rfv = torch.zeros_like(self.U)
            self.fv_list = torch.zeros(max(d.ne, 1), dtype=torch.int32, device=self.dev)
            self.fv_count = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._fill_desc()

    def ensure_gradients(self):
        d = self.d
        if self.g is None and d.viscous:
            f64 = dict(dtype=self.torch.float64, device=self.dev)
            n1 = d.n1
            self.g = self.torch.zeros((d.ne, n1, n1, n1, 3, N_LIFT), **f64)
            self.gL = self.torch.zeros((d.ns, n1, n1, 3, N_LIFT), **f64)
            self.gR = self.torch.zeros((d.ns, n1, n1, 3, N_LIFT), **f64)
            self.vstar = self.torch.zeros((d.ns, n1, n1, N_LIFT), **f64)
            self._fill_desc()

    def drop_gradients(self):
        self.g = self.gL = self.gR = self.vstar = None
        self._fill_desc()

    def download_gradients(self):
        d = self.d
        if self.g is None:
            return
        d.g[...] = self.g.cpu().numpy()
        d.gL[...] = self.gL.cpu().numpy()
        d.gR[...] = self.gR.cpu().numpy()
        d.vstar[...] = self.vstar.cpu().numpy()

    def upload_state(self):
        self.U.copy_(self.torch.as_tensor(self.d.U))
        self.upload_bc()
        self.dt_valid = False   # dt_bits no longer holds the local dt of this U

    def upload_bc(self):
        self.bc.copy_(self.torch.as_tensor(np.ascontiguousarray(self.d.bc_states)))

    def upload_traces(self, from_host=False):
        if from_host:
            self.UL.copy_(self.torch.as_tensor(self.d.UL))
            self.UR.copy_(self.torch.as_tensor(self.d.UR))

    def local_dt(self, U, cfl, cfl_visc, prm):
        """Device k_local_dt; returns the host float (syncs)."""
        self.dt_bits.fill_(0x7FF0000000000000)
        self.status.copy_(self.status_init)
        _lib.check(self.lib.hdg_local_dt(self.dptr, ctypes.byref(prm), _lib.ptr(U), cfl, cfl_visc,
                                         self.sptr()), "hdg_local_dt")
        bits = self.dt_bits.cpu().numpy()[:1].copy()
        return float(bits.view(np.float64)[0])
