"""Multi-GPU SPIKE: one slab of rows per GPU, two-level reduced system.

The production data plane is C++ (paper_1811_03559_b200/csrc/spk_dist.cu:
spk_comm_* / spk_dist_factorize / spk_dist_solve, NCCL all-gathers issued by
the library on the caller's stream); :class:`NcclPlane` below wires it to a
torch.distributed process group (the NCCL unique id travels over the group).
The generator protocol in this module is the same algorithm written over
torch tensors: the CPU (gloo) tests and the one-GPU virtual-rank tests run it,
and the GPU tests check the C++ exchange arithmetic against it.

SURVEY.md section 8(e).  The reference has no multi-GPU path (it is a
single-node fork-join library, ``proj/include/spike/parallel_util.hpp:13-45``);
this module extends its algorithm along the line the paper's recursive
reduction already draws: each GPU factors its slab as a SPIKE system of its own
(``spk_factorize_slab``), whose edge partitions also carry the spikes coupling
them to the neighbouring slabs, and collapses its reduced hierarchy into ONE
unit.  The G slab units form a reduced system of exactly the reference's shape
(``reduce_factorize``, ``factorize.cpp:46-120``) with p = G, held redundantly
on every GPU.

Exchanges (device tensors, all tiny next to the slab work):

* factorize: all-gather of each slab unit's tips [vt; vb; wt; wb] (4 k*k).
* solve: all-gather of [y_top; y_bot] (2k x nrhs); slab-level reduced solve;
  each GPU corrects its reduced rows with its unit spikes and retrieves.
* transpose solve: all-gather of the edge G-tip terms (2k x nrhs), then of
  [t_top; t_bot; V_int^T t; W_int^T t] (4k x nrhs); slab-level transposed
  reduced solve; local transposed reduction and D^T stage.

The per-rank protocol is a generator that yields its export block and
receives the gathered blocks of all ranks, so the same code runs under
``torch.distributed`` (one process per GPU, NCCL) via :func:`collective` and,
for tests, as G virtual ranks in one process via :func:`lockstep`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Generator, List, Optional, Sequence

import torch

from . import spike as _spk
from .spike import FactorOptions, PartitionPlan, _check, _Opts, _plan_struct, lib


# ----------------------------------------------------------------------------
# geometry
def slab_rows(n: int, world: int) -> List[int]:
    """Row boundaries of `world` equal slabs (first `n % world` one row longer)."""
    if world < 1 or n < world:
        raise _spk.InvalidArgument("slab_rows: need 1 <= world <= n")
    base, extra = divmod(n, world)
    b = [0]
    for g in range(world):
        b.append(b[-1] + base + (1 if g < extra else 0))
    return b


def halo(rank: int, world: int, k: int):
    """(left, right) halo columns of a slab: k per open edge."""
    return (k if rank > 0 else 0), (k if rank < world - 1 else 0)


def load_slab_band(path, rank: int, world: int, device=None, stream: int = 0):
    """This rank's slab of a .spkb band straight into HBM (spk_spkb_load): the
    packed columns [R_g - left halo, R_{g+1} + right halo), i.e. the band
    spk_factorize_slab takes; no other rank's rows are read.  Returns
    (tensor (ncols, kl+ku+1), (n, kl, ku), left halo)."""
    n, kl, ku = _spk.spkb_header(path)
    k = max(kl, ku)
    rows = slab_rows(n, world)
    lh, rh = halo(rank, world, k)
    c0 = rows[rank] - lh
    nc = rows[rank + 1] - rows[rank] + lh + rh
    t = torch.empty((nc, kl + ku + 1), dtype=torch.float64, device=device or torch.device("cuda"))
    _spk.load_spkb_device(path, t.data_ptr(), c0, nc, stream)
    return t, (n, kl, ku), lh


# ----------------------------------------------------------------------------
# slab-level reduced-system assembly (pure tensor code: device or CPU)
def gather_tips_host(gathered: torch.Tensor, k: int):
    """(G, 4k^2) gathered unit tips -> four contiguous (G, k^2) float64 host
    arrays vt, vb, wt, wb (column-major k x k blocks, spk_reduced_create)."""
    h = gathered.reshape(gathered.shape[0], 4, k * k).to("cpu", torch.float64)
    return [h[:, q, :].contiguous().numpy() for q in range(4)]


def forward_top_rhs(gathered: torch.Tensor, k: int, nrhs: int) -> torch.Tensor:
    """(G, 2k*nrhs) exports [y_top; y_bot] -> slab-level reduced RHS as an
    (nrhs, 2Gk) tensor = column-major 2Gk x nrhs."""
    G = gathered.shape[0]
    return gathered.reshape(G, nrhs, 2 * k).permute(1, 0, 2).reshape(nrhs, 2 * G * k).contiguous()


def forward_import(z: torch.Tensor, rank: int, world: int, k: int) -> torch.Tensor:
    """Solved tips (nrhs, 2Gk) -> this slab's import [xi; eta]: the right
    slab's x_top and the left slab's x_bot (zero at closed edges)."""
    nrhs = z.shape[0]
    zt = z.reshape(nrhs, world, 2, k)
    imp = torch.zeros(nrhs, 2, k, dtype=z.dtype, device=z.device)
    if rank + 1 < world:
        imp[:, 0] = zt[:, rank + 1, 0]
    if rank > 0:
        imp[:, 1] = zt[:, rank - 1, 1]
    return imp.reshape(nrhs, 2 * k).contiguous()


def transpose_import1(gathered: torch.Tensor, rank: int, world: int, k: int, nrhs: int) -> torch.Tensor:
    """(G, 2k*nrhs) exports [chat_0^T tau_t; bhat_last^T tau_b] -> this slab's
    [left slab's bhat^T tau_b; right slab's chat^T tau_t]."""
    a = gathered.reshape(world, nrhs, 2, k)
    imp = torch.zeros(nrhs, 2, k, dtype=gathered.dtype, device=gathered.device)
    if rank > 0:
        imp[:, 0] = a[rank - 1, :, 1]
    if rank + 1 < world:
        imp[:, 1] = a[rank + 1, :, 0]
    return imp.reshape(nrhs, 2 * k).contiguous()


def transpose_top_rhs(gathered: torch.Tensor, k: int, nrhs: int) -> torch.Tensor:
    """(G, 4k*nrhs) exports [t_top; t_bot; c; d] -> RHS of S_G^T z = t - C^T t_int
    as (nrhs, 2Gk): top(h) -= c(h-1) (left slab's V_int^T t), bot(h) -= d(h+1)."""
    G = gathered.shape[0]
    b = gathered.reshape(G, nrhs, 4, k).permute(1, 0, 2, 3)  # (nrhs, G, 4, k)
    rhs = b[:, :, 0:2, :].clone()
    if G > 1:
        rhs[:, 1:, 0] -= b[:, :-1, 2]
        rhs[:, :-1, 1] -= b[:, 1:, 3]
    return rhs.reshape(nrhs, 2 * G * k).contiguous()


def transpose_import2(z: torch.Tensor, rank: int, world: int, k: int) -> torch.Tensor:
    nrhs = z.shape[0]
    return z.reshape(nrhs, world, 2, k)[:, rank].reshape(nrhs, 2 * k).contiguous()


# ----------------------------------------------------------------------------
# per-rank protocols
Exchange = Generator[torch.Tensor, torch.Tensor, object]


def factorize_steps(slab, boost_eps: float) -> Exchange:
    """Factor the slab, exchange unit tips, factor the slab-level system.
    Returns (slab, top)."""
    tips = slab.factor_tips()
    gathered = yield tips
    top = slab.top_create(gathered, boost_eps)
    return slab, top


def solve_steps(slab, top, transpose: bool) -> Exchange:
    """One solve (or transpose solve) of the global system; X written in place."""
    k, g, G, nrhs = slab.k, slab.rank, slab.world, slab.nrhs
    state, exp = slab.begin(transpose)
    if not transpose:
        gathered = yield exp
        z = forward_top_rhs(gathered, k, nrhs)
        slab.top_solve(top, False, z)
        slab.step(state, forward_import(z, g, G, k))
    else:
        gathered = yield exp
        exp2 = slab.step(state, transpose_import1(gathered, g, G, k, nrhs))
        gathered = yield exp2
        z = transpose_top_rhs(gathered, k, nrhs)
        slab.top_solve(top, True, z)
        slab.step(state, transpose_import2(z, g, G, k))
    slab.end(state)
    return None


# ----------------------------------------------------------------------------
# drivers
def collective(gen: Exchange, group=None):
    """Run a per-rank protocol under torch.distributed (NCCL for CUDA tensors,
    gloo for CPU tensors): every yield is an all-gather."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    try:
        out = next(gen)
        while True:
            parts = [torch.empty_like(out) for _ in range(world)]
            dist.all_gather(parts, out.contiguous(), group=group)
            out = gen.send(torch.stack(parts))
    except StopIteration as e:
        return e.value


def lockstep(gens: Sequence[Exchange]):
    """Run G per-rank protocols in one process (virtual ranks): every yield is
    a concatenation.  For tests on one GPU; no rank waits on another."""
    outs = [next(g) for g in gens]
    results: List[object] = [None] * len(gens)
    done = [False] * len(gens)
    while not all(done):
        stacked = torch.stack([o for o in outs])
        for i, g in enumerate(gens):
            try:
                outs[i] = g.send(stacked)
            except StopIteration as e:
                results[i] = e.value
                done[i] = True
        if any(done) and not all(done):
            raise RuntimeError("lockstep: ranks disagree on the number of exchanges")
    return results


# ----------------------------------------------------------------------------
# the CUDA slab (C-ABI: spk_factorize_slab / spk_xsolve_*)
class _Top:
    def __init__(self, h, world, k):
        self.h, self.world, self.k = h, world, k

    def __del__(self):
        try:
            if self.h:
                lib().spk_reduced_destroy(self.h)
        except Exception:
            pass


class CudaSlab:
    """Rows [row0, row0 + n) of the global system on the current CUDA device.

    band_ptr addresses the slab's packed band including its halo columns
    (k per open edge, ``halo``); the plan partitions the slab's own rows."""

    def __init__(self, band_ptr: int, n: int, kl: int, ku: int, plan: PartitionPlan, rank: int, world: int,
                 opts: Optional[FactorOptions] = None, stream: Optional[int] = None):
        self.band_ptr, self.n, self.kl, self.ku = band_ptr, n, kl, ku
        self.k = max(kl, ku)
        self.plan, self.rank, self.world = plan, rank, world
        self.opts = opts or FactorOptions()
        self.stream = torch.cuda.current_stream().cuda_stream if stream is None else stream
        self.fact = None
        self.nrhs = 0
        self._io = None

    # factorize
    def factor_tips(self) -> torch.Tensor:
        st, keep = _plan_struct(self.plan)
        o = _Opts(int(bool(self.opts.pivoting)), float(self.opts.boost_eps))
        h = C.c_void_p()
        _check(lib().spk_factorize_slab(C.c_void_p(self.band_ptr), 1, self.n, self.kl, self.ku, C.byref(st),
                                        C.byref(o), int(self.rank > 0), int(self.rank < self.world - 1),
                                        C.c_void_p(self.stream), C.byref(h)))
        self.fact = _spk.SpikeFactorization(h.value, self.plan, self.n, self.kl, self.ku, self.opts)
        tips = torch.empty(4 * self.k * self.k, dtype=torch.float64, device="cuda")
        _check(lib().spk_fact_unit_tips(self.fact._h, C.c_void_p(tips.data_ptr()), C.c_void_p(self.stream)))
        return tips

    def top_create(self, gathered: torch.Tensor, boost_eps: float) -> _Top:
        # the gathered (G, 4k^2) tips stay in HBM: assembled and factored on the device
        g = gathered.contiguous()
        h = C.c_void_p()
        _check(lib().spk_reduced_create_device(C.c_void_p(g.data_ptr()), self.world, self.k, boost_eps,
                                               C.c_void_p(self.stream), C.byref(h)))
        return _Top(h.value, self.world, self.k)

    def top_solve(self, top: _Top, transpose: bool, z: torch.Tensor) -> None:
        _check(lib().spk_reduced_solve_device(top.h, int(transpose), C.c_void_p(z.data_ptr()), z.shape[0],
                                              C.c_void_p(self.stream)))

    # solve: bind the right-hand sides, then run solve_steps
    def bind(self, f_ptr: int, ldf: int, nrhs: int, x_ptr: int, ldx: int):
        self._io = (f_ptr, ldf, x_ptr, ldx)
        self.nrhs = nrhs

    def begin(self, transpose: bool):
        f_ptr, ldf, x_ptr, ldx = self._io
        exp = torch.empty(2 * self.k * self.nrhs, dtype=torch.float64, device="cuda")
        h = C.c_void_p()
        _check(lib().spk_xsolve_begin(self.fact._h, int(transpose), C.c_void_p(f_ptr), ldf, self.nrhs,
                                      C.c_void_p(x_ptr), ldx, C.c_void_p(self.stream), C.c_void_p(exp.data_ptr()),
                                      C.byref(h)))
        return [h.value, transpose, 0], exp

    def step(self, state, imp: torch.Tensor):
        h, transpose, q = state
        state[2] += 1
        exp = None
        if transpose and q == 0:
            exp = torch.empty(4 * self.k * self.nrhs, dtype=torch.float64, device="cuda")
        _check(lib().spk_xsolve_step(C.c_void_p(h), C.c_void_p(imp.data_ptr()),
                                     C.c_void_p(exp.data_ptr() if exp is not None else None)))
        return exp

    def end(self, state):
        lib().spk_xsolve_end(C.c_void_p(state[0]))


@dataclass
class DistributedFactorization:
    slab: CudaSlab
    top: _Top


def factorize_distributed(band_ptr: int, n_local: int, kl: int, ku: int, plan: PartitionPlan,
                          opts: Optional[FactorOptions] = None, group=None) -> DistributedFactorization:
    """Collective over the process group: this rank's slab (band with halo
    columns, see ``halo``) is factored and the slab-level system assembled."""
    import torch.distributed as dist

    opts = opts or FactorOptions()
    slab = CudaSlab(band_ptr, n_local, kl, ku, plan, dist.get_rank(group), dist.get_world_size(group), opts)
    slab, top = collective(factorize_steps(slab, opts.boost_eps), group)
    return DistributedFactorization(slab, top)


def solve_distributed(df: DistributedFactorization, f_ptr: int, ldf: int, nrhs: int, x_ptr: int, ldx: int,
                      transpose: bool = False, group=None) -> None:
    """Collective: this rank's rows of X := A^-1 F (or A^-T F)."""
    if df.slab.world == 1:
        _spk.solve_device(df.slab.fact, f_ptr, ldf, nrhs, x_ptr, ldx, transpose, df.slab.stream)
        return
    df.slab.bind(f_ptr, ldf, nrhs, x_ptr, ldx)
    collective(solve_steps(df.slab, df.top, transpose), group)


# ----------------------------------------------------------------------------
# the C++ data plane (spk_dist.cu)
def exchange_device(op: int, src: torch.Tensor, G: int, rank: int, k: int, nrhs: int, stream: int = 0) -> torch.Tensor:
    """spk_dist_exchange: the library's exchange arithmetic (ops SPK_XCH_*),
    returned as a flat device tensor."""
    n_out = 2 * G * k * nrhs if op in (XCH_FWD_TOP_RHS, XCH_TR_TOP_RHS) else 2 * k * nrhs
    dst = torch.empty(n_out, dtype=torch.float64, device=src.device)
    _spk._dcheck(lib().spk_dist_exchange(op, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), G, rank, k,
                                         nrhs, C.c_void_p(stream)))
    return dst


XCH_FWD_TOP_RHS, XCH_FWD_IMPORT, XCH_TR_IMPORT1, XCH_TR_TOP_RHS, XCH_TR_IMPORT2 = range(5)


class NcclPlane:
    """One rank of the C++ multi-GPU data plane: an NCCL communicator owned by
    the library (its unique id broadcast over the torch.distributed group),
    slab factorizations and solves whose tip exchanges the library issues
    itself on the caller's stream."""

    ID_BYTES = 128

    def __init__(self, group=None, rank: Optional[int] = None, world: Optional[int] = None):
        import torch.distributed as dist

        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        uid = torch.zeros(self.ID_BYTES, dtype=torch.uint8)
        if self.rank == 0:
            buf = (C.c_uint8 * self.ID_BYTES)()
            _spk._dcheck(lib().spk_comm_unique_id(buf))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if self.world > 1:
            dev_uid = uid.to("cuda") if dist.get_backend(group) == "nccl" else uid
            dist.broadcast(dev_uid, 0, group=group)
            uid = dev_uid.cpu()
        raw = (C.c_uint8 * self.ID_BYTES)(*uid.tolist())
        h = C.c_void_p()
        _spk._dcheck(lib().spk_comm_init(raw, self.world, self.rank, C.byref(h)))
        self.h = h.value

    @classmethod
    def single(cls):
        """A one-rank plane (no process group): the data plane's G = 1 case."""
        self = cls.__new__(cls)
        self.rank, self.world = 0, 1
        buf = (C.c_uint8 * cls.ID_BYTES)()
        _spk._dcheck(lib().spk_comm_unique_id(buf))
        h = C.c_void_p()
        _spk._dcheck(lib().spk_comm_init(buf, 1, 0, C.byref(h)))
        self.h = h.value
        return self

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().spk_comm_destroy(C.c_void_p(self.h))
        except Exception:
            pass

    def factorize(self, band_ptr: int, n_local: int, kl: int, ku: int, plan: PartitionPlan,
                  opts: Optional[FactorOptions] = None, stream: int = 0) -> "DistFact":
        opts = opts or FactorOptions()
        st, keep = _plan_struct(plan)
        o = _Opts(int(bool(opts.pivoting)), float(opts.boost_eps))
        h = C.c_void_p()
        _spk._dcheck(lib().spk_dist_factorize(C.c_void_p(band_ptr), n_local, kl, ku, C.byref(st), C.byref(o),
                                              C.c_void_p(self.h), C.c_void_p(stream), C.byref(h)))
        return DistFact(h.value, self)

    def solve(self, df: "DistFact", f_ptr: int, ldf: int, nrhs: int, x_ptr: int, ldx: int,
              transpose: bool = False, stream: int = 0) -> None:
        _spk._dcheck(lib().spk_dist_solve(C.c_void_p(df.h), int(transpose), C.c_void_p(f_ptr), ldf, nrhs,
                                          C.c_void_p(x_ptr), ldx, C.c_void_p(stream)))


class DistFact:
    def __init__(self, h, plane):
        self.h, self.plane = h, plane

    def __del__(self):
        try:
            if self.h:
                lib().spk_dist_destroy(C.c_void_p(self.h))
        except Exception:
            pass
