"""Dynamic Axial Parallelism (DAP) over torch.distributed / NCCL.

Reference: dap_block.py:46-152 (the sharded schedule), sharding.py:26-212
(mesh, ledger, collective semantics) and commcost.py:126-158 (the byte-exact
ledger prediction).  The reference simulates devices as a Python loop; here
one process drives one GPU and the collectives are real:

  reference (simulated)                 here
  all_to_all_switch_axis (sharding:130)  dist.all_to_all_single (pack-free on one side)
  all_gather (sharding:162)              dist.all_gather_into_tensor, rank-major output
                                         addressed in place by the GEMMs (no unpack)
  (no backward in the reference)         all-gather^T = reduce_scatter_tensor, a2a^T = a2a

Canonical shards (dap_block.py:58-59, 150-151): m on the sequence axis,
z on the row axis; blocks chain on shards.  Per block forward: 6 all-to-all,
3 projection all-gathers, 1 bias all-gather (ledger categories as the
reference's CommLedger).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import torch

from .config import EvoConfig
from .errors import DomainError, MeshError, ShardError

REPORTING_ELEMENT_SIZE = 2


# ----------------------------------------------------------------------------- mesh + ledger
@dataclass(frozen=True)
class DeviceMesh:
    """1-D mesh (sharding.py:26-44).  On the GPU path device d is torch.distributed rank d;
    device_order only permutes host-side iteration and never changes results."""

    n_devices: int
    device_order: tuple = ()

    def __post_init__(self):
        if self.n_devices < 1:
            raise MeshError(f"need at least one device, got {self.n_devices}")
        order = self.device_order or tuple(range(self.n_devices))
        if sorted(order) != list(range(self.n_devices)):
            raise MeshError(f"device_order {order} is not a permutation of range({self.n_devices})")
        object.__setattr__(self, "device_order", tuple(order))


class CommLedger:
    """Per-device, per-category collective traffic (sharding.py:47-92), same JSON schema
    ``evoplan-ledger-v1``.  Bytes are logical sends under the reporting element size."""

    def __init__(self, n_devices: int, element_size: int = REPORTING_ELEMENT_SIZE):
        self.n_devices = n_devices
        self.element_size = element_size
        self.counts: dict[str, int] = {}
        self.bytes: dict[str, list[int]] = {}

    def record(self, category: str, per_device_elements) -> None:
        if len(per_device_elements) != self.n_devices:
            raise MeshError("ledger entry must cover every device")
        self.counts[category] = self.counts.get(category, 0) + 1
        row = self.bytes.setdefault(category, [0] * self.n_devices)
        for d, e in enumerate(per_device_elements):
            row[d] += int(e) * self.element_size

    def total_bytes(self, category: str | None = None) -> int:
        if category is not None:
            return sum(self.bytes.get(category, []))
        return sum(sum(v) for v in self.bytes.values())

    def device_bytes(self, device: int) -> int:
        return sum(v[device] for v in self.bytes.values())

    def summary(self) -> dict:
        return {cat: {"count": self.counts[cat], "bytes": sum(self.bytes[cat])} for cat in self.counts}

    def to_json(self) -> str:
        per_device = [{cat: {"count": self.counts[cat], "bytes": self.bytes[cat][d]} for cat in sorted(self.counts)}
                      for d in range(self.n_devices)]
        totals = {cat: {"count": self.counts[cat], "bytes": sum(self.bytes[cat])} for cat in sorted(self.counts)}
        return json.dumps({"schema": "evoplan-ledger-v1", "n_devices": self.n_devices,
                           "element_size": self.element_size, "per_device": per_device, "totals": totals},
                          sort_keys=True)


def predict_block_ledger(cfg: EvoConfig, n_devices: int, element_size: int = 2) -> dict:
    """Expected forward ledger of one sharded block (commcost.py:126-158): count and total
    bytes summed over devices for all_to_all / all_gather / bias_gather."""
    if n_devices < 1:
        raise DomainError(f"device count must be positive, got {n_devices}")
    if n_devices == 1:
        return {}
    es, n = element_size, n_devices
    m_bytes = cfg.n_seq * cfg.n_res * cfg.h_msa * es
    z_bytes = cfg.n_res * cfg.n_res * cfg.h_pair * es
    opm_factor = cfg.n_seq * cfg.n_res * cfg.hidden_proj * es
    tri_factor = cfg.n_res * cfg.n_res * cfg.hidden_proj * es
    bias_bytes = cfg.n_res * cfg.n_res * cfg.n_head_msa * es
    return {
        "all_to_all": {"count": 6, "bytes": round((2 * m_bytes + 4 * z_bytes) * (n - 1) / n)},
        "all_gather": {"count": 3, "bytes": round((opm_factor + 2 * tri_factor) * (n - 1))},
        "bias_gather": {"count": 1, "bytes": round(bias_bytes * (n - 1))},
    }


# ----------------------------------------------------------------------------- communicators
class DapComm:
    """Collectives of one DAP rank over a torch.distributed process group (NCCL on the GPU,
    gloo in the host-logic tests).  Every call records the reference's ledger categories;
    backward collectives use their own categories ("reduce_scatter", "grad_all_reduce").

    Buffers are rank-major: all_gather(t) -> [N, *t.shape]; all_to_all(t [N, ...]) sends
    chunk d to rank d and returns [N(src), ...]; reduce_scatter(t [N, ...]) -> sum over
    ranks of chunk `rank`."""

    def __init__(self, group=None, ledger: CommLedger | None = None, overlap: bool = True):
        """overlap: asynchronous collectives (DAO) - the projection all-gathers,
        the backward reduce-scatters and the gradient all-reduce run on the communicator's stream
        under independent compute.  overlap=False issues the same collectives synchronously (same
        buffers, same order, same bits: tests/test_dap_gloo.py compares the two schedules)."""
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.overlap = overlap
        if dist.is_available() and dist.is_initialized():
            self.N = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.N, self.rank = 1, 0
        self.ledger = ledger

    def _rec(self, category, elems):
        if self.ledger is not None:
            self.ledger.record(category, [elems] * self.N)

    def all_gather(self, t, category="all_gather", async_op=False):
        """-> out [N, *t.shape]  (or (out, handle) with async_op: call handle.wait() before use)"""
        t = t.contiguous()
        out = torch.empty((self.N,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if self.N == 1:
            out[0].copy_(t)
            return (out, _Done()) if async_op else out
        # concatenated-along-dim-0 form (accepted by NCCL and gloo); same memory as [N, ...]
        work = self.dist.all_gather_into_tensor(out.view((self.N * t.shape[0],) + tuple(t.shape[1:])), t,
                                                group=self.group, async_op=async_op)
        self._rec(category, t.numel() * (self.N - 1))
        return (out, work) if async_op else out

    def reduce_scatter(self, t, category="reduce_scatter", async_op=False):
        """sum over ranks of chunk `rank` of t [N, ...]; async_op: returns a zero-argument callable
        that waits and returns the result (the caller runs independent work in between)."""
        t = t.contiguous()
        if self.N == 1:
            return (lambda: t[0]) if async_op else t[0]
        out = torch.empty(tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        work = self.dist.reduce_scatter_tensor(out, t.flatten(0, 1), op=self.dist.ReduceOp.SUM, group=self.group,
                                               async_op=async_op and self.overlap)
        self._rec(category, t[0].numel() * (self.N - 1))
        if not async_op:
            return out
        if work is None:
            return lambda: out

        def finish():
            work.wait()
            return out
        return finish

    def gather_fn(self, category="all_gather"):
        """the ``gather`` callable block.py takes: gather(t) -> [N, *t.shape]; gather(t, async_op=True)
        -> zero-argument callable returning it after the collective completed"""
        def gather(t, async_op=False):
            if not async_op:
                return self.all_gather(t, category)
            if not self.overlap:
                out = self.all_gather(t, category)
                return lambda: out
            out, work = self.all_gather(t, category, async_op=True)

            def finish():
                work.wait()
                return out
            return finish
        return gather

    def reduce_scatter_fn(self, category="reduce_scatter"):
        return lambda t, async_op=False: self.reduce_scatter(t, category, async_op=async_op)

    def all_to_all(self, t, category="all_to_all", async_op=False):
        t = t.contiguous()
        if self.N == 1:
            return (t, _Done()) if async_op else t
        out = torch.empty_like(t)
        work = self.dist.all_to_all_single(out, t, group=self.group, async_op=async_op)
        self._rec(category, t.numel() - t.numel() // self.N)
        return (out, work) if async_op else out

    def all_reduce_(self, t, category="grad_all_reduce", async_op=False):
        """in-place sum over ranks; async_op: returns a handle with wait() (the gradient all-reduce
        of block i runs under block i-1's backward)"""
        if self.N == 1:
            return _Done() if async_op else t
        work = self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group,
                                    async_op=async_op and self.overlap)
        self._rec(category, 2 * t.numel() * (self.N - 1) // self.N)
        if async_op:
            return work if work is not None else _Done()
        return t

    def all_reduce_max(self, x: float) -> float:
        if self.N == 1:
            return x
        t = torch.tensor([x], device="cuda" if torch.cuda.is_available() else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class _Done:
    """handle of an already-completed collective"""

    def wait(self):
        return None


class ThreadMesh:
    """N virtual DAP ranks inside ONE process (one Python thread per rank, sharing the
    GPU).  Used by ``dap_evoformer_block`` when no process group of the mesh's size
    exists - the reference's single-process simulation (dap_block.py:39-43), but with
    the real kernels and the same SPMD schedule as the NCCL path.  Collectives are
    rendezvous through shared slots + a barrier (device-synchronised)."""

    def __init__(self, n: int):
        import threading
        self.n = n
        self.barrier = threading.Barrier(n)
        self.slots: list = [None] * n

    def exchange(self, rank: int, value):
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        self.slots[rank] = value
        self.barrier.wait()
        got = list(self.slots)
        self.barrier.wait()
        return got


class ThreadComm(DapComm):
    def __init__(self, mesh: ThreadMesh, rank: int, ledger: CommLedger | None = None):
        self.mesh, self.N, self.rank, self.ledger = mesh, mesh.n, rank, ledger
        self.group = None
        self.overlap = False  # rendezvous collectives complete on return

    def _rec(self, category, elems):
        # one ledger shared by the virtual ranks: rank 0 records for all (symmetric shards)
        if self.ledger is not None and self.rank == 0:
            self.ledger.record(category, [elems] * self.N)

    def all_gather(self, t, category="all_gather", async_op=False):
        parts = self.mesh.exchange(self.rank, t.contiguous())
        if self.N > 1:
            self._rec(category, t.numel() * (self.N - 1))
        out = torch.stack(parts, 0)
        return (out, _Done()) if async_op else out

    def reduce_scatter(self, t, category="reduce_scatter", async_op=False):
        parts = self.mesh.exchange(self.rank, t.contiguous())
        if self.N > 1:
            self._rec(category, t[0].numel() * (self.N - 1))
        out = parts[0][self.rank].clone()
        for p in parts[1:]:
            out += p[self.rank]
        return (lambda: out) if async_op else out

    def all_to_all(self, t, category="all_to_all", async_op=False):
        parts = self.mesh.exchange(self.rank, t.contiguous())
        if self.N > 1:
            self._rec(category, t.numel() - t.numel() // self.N)
        out = torch.stack([p[self.rank] for p in parts], 0)
        return (out, _Done()) if async_op else out

    def all_reduce_(self, t, category="grad_all_reduce", async_op=False):
        parts = self.mesh.exchange(self.rank, t.clone())
        if self.N > 1:
            self._rec(category, 2 * t.numel() * (self.N - 1) // self.N)
        t.copy_(sum(parts[1:], parts[0]))
        return _Done() if async_op else t

    def all_reduce_max(self, x: float) -> float:
        return max(self.mesh.exchange(self.rank, x))


# ----------------------------------------------------------------------------- axis switches
def switch_rows_to_cols(comm: DapComm, x, async_op=False):
    """[A/N, Bf, C] sharded on axis 0 -> [A, Bf/N, C] sharded on axis 1
    (all_to_all_switch_axis(t, 1), sharding.py:130-159).  The send side packs the
    destination-major buffer; the received rank-major buffer IS the result."""
    N = comm.N
    if N == 1:
        return (lambda: x) if async_op else x
    Al, Bf, C = x.shape
    if Bf % N:
        raise ShardError(f"extent {Bf} on axis 1 not divisible by {N} devices")
    send = x.view(Al, N, Bf // N, C).permute(1, 0, 2, 3)
    if async_op:
        recv, work = comm.all_to_all(send, async_op=True)

        def finish():
            work.wait()
            return recv.view(N * Al, Bf // N, C)
        return finish
    return comm.all_to_all(send).view(N * Al, Bf // N, C)


def switch_cols_to_rows(comm: DapComm, x, async_op=False):
    """[A, Bl, C] sharded on axis 1 -> [A/N, Bl*N, C] sharded on axis 0.  The send
    buffer is x itself (chunks along axis 0 are contiguous); the receive side unpacks.
    async_op: returns a zero-argument callable that waits and unpacks (DAO overlap)."""
    N = comm.N
    if N == 1:
        return (lambda: x) if async_op else x
    A, Bl, C = x.shape
    if A % N:
        raise ShardError(f"extent {A} on axis 0 not divisible by {N} devices")
    if async_op:
        recv, work = comm.all_to_all(x.view(N, A // N, Bl, C), async_op=True)

        def finish():
            work.wait()
            return recv.permute(1, 0, 2, 3).reshape(A // N, N * Bl, C)
        return finish
    recv = comm.all_to_all(x.view(N, A // N, Bl, C))
    return recv.permute(1, 0, 2, 3).reshape(A // N, N * Bl, C)


# ----------------------------------------------------------------------------- the DAP block
def dap_block_fwd(bp, comm: DapComm, m_loc, z_loc, save=True):
    """One Evoformer block on this rank's canonical shards (dap_block.py:46-152):
    m_loc [N_s/N, N_r, H_m] (sequence shard), z_loc [N_r/N, N_r, H_z] (row shard).
    Returns the updated canonical shards and the saved context."""
    from . import block as B
    cfg = bp.cfg
    N = comm.N
    S, R, Hm, Hz = cfg.n_seq, cfg.n_res, cfg.h_msa, cfg.h_pair
    if S % N or R % N:
        raise ShardError(f"n_seq={S} / n_res={R} not divisible by {N} devices")
    Sl, Rl = S // N, R // N
    nh = cfg.n_head_msa
    sv = {}
    # 1) pair-derived row-attention bias from local pair rows, gathered (dap_block.py:63-64)
    bias_loc, sv["bias"] = B.msa_row_bias_fwd(bp, z_loc.reshape(Rl * R, Hz), Rl, R, save)
    # DAO: the gather runs on NCCL's stream while msa_row's LN + q/k/v/g GEMMs run here
    g, work = comm.all_gather(bias_loc, "bias_gather", async_op=True)    # [N, nh, Rl, R]

    def bias_ready():
        work.wait()
        return g.permute(1, 0, 2, 3).reshape(nh, R, R) if N > 1 else g[0]
    m2, sv["msa_row"] = B.attention_fwd(bp, "msa_row", m_loc.reshape(Sl * R, Hm), Sl, R, "row", bias=bias_ready,
                                        save=save)
    # 2) sequence shard -> residue shard (dap_block.py:69)
    m_r = switch_rows_to_cols(comm, m2.view(Sl, R, Hm))               # [S, Rl, Hm]
    m2, sv["msa_col"] = B.attention_fwd(bp, "msa_col", m_r.reshape(S * Rl, Hm), Rl, S, "col", save=save)
    m2, sv["msa_trans"] = B.transition_fwd(bp, "msa_trans", m2, S * Rl, save)
    # DAO: m is final here; its switch back to the sequence shard overlaps the pair stack
    m_out_ready = None  # issued after the OPM (which still reads m2)
    # 3) outer product mean: right projection gathered (dap_block.py:81-94)
    gat = comm.gather_fn() if N > 1 else None
    z2, sv["opm"] = B.opm_fwd(bp, m2, z_loc.reshape(Rl * R, Hz), S, Rl, save, gather=gat)
    m_out_ready = switch_cols_to_rows(comm, m2.view(S, Rl, Hm), async_op=True)
    # 4) outgoing triangle: b gathered across the row shard (dap_block.py:98-111)
    z2, sv["tri_out"] = B.triangle_fwd(bp, "tri_out", z2, R, save, Rl=Rl, gather=gat)
    # 5) row shard -> column shard, incoming triangle gathers a (dap_block.py:114-128)
    z_c = switch_rows_to_cols(comm, z2.view(Rl, R, Hz))               # [R, Rl, Hz]
    z2, sv["tri_in"] = B.triangle_fwd(bp, "tri_in", z_c.reshape(R * Rl, Hz), R, save, Rl=Rl, gather=gat)
    # 6) column -> row shard, pair row attention (dap_block.py:131-135)
    z_r = switch_cols_to_rows(comm, z2.view(R, Rl, Hz))               # [Rl, R, Hz]
    z2, sv["pair_row"] = B.attention_fwd(bp, "pair_row", z_r.reshape(Rl * R, Hz), Rl, R, "row", bias="pair",
                                         save=save)
    # 7) row -> column shard, pair column attention + transition (dap_block.py:138-147)
    z_c = switch_rows_to_cols(comm, z2.view(Rl, R, Hz))
    z2, sv["pair_col"] = B.attention_fwd(bp, "pair_col", z_c.reshape(R * Rl, Hz), Rl, R, "col", bias="pair",
                                         save=save)
    z2, sv["pair_trans"] = B.transition_fwd(bp, "pair_trans", z2, R * Rl, save)
    # 8) restore canonical shards (dap_block.py:150-151)
    z_out = switch_cols_to_rows(comm, z2.view(R, Rl, Hz))             # [Rl, R, Hz]
    m_out = m_out_ready()                                             # [Sl, R, Hm]
    return m_out.contiguous(), z_out.contiguous(), (sv if save else None)


def dap_block_bwd(bp, comm: DapComm, sv, dm_loc, dz_loc):
    """Backward of dap_block_fwd: every all-to-all is inverted, every all-gather becomes a
    reduce-scatter of the partial gradients of the gathered factor.  Parameter gradients
    are this rank's partial sums (all-reduce them across ranks once per step)."""
    from . import block as B
    cfg = bp.cfg
    N = comm.N
    S, R, Hm, Hz = cfg.n_seq, cfg.n_res, cfg.h_msa, cfg.h_pair
    Sl, Rl = S // N, R // N
    nh = cfg.n_head_msa
    rs = comm.reduce_scatter_fn() if N > 1 else None
    dm_r_ready = switch_rows_to_cols(comm, dm_loc.view(Sl, R, Hm), async_op=True)  # overlaps the pair stack
    dz_c = switch_rows_to_cols(comm, dz_loc.view(Rl, R, Hz))          # inverse of step 8
    dz2 = B.transition_bwd(bp, sv["pair_trans"], dz_c.reshape(R * Rl, Hz).contiguous())
    dz2, _ = B.attention_bwd(bp, sv["pair_col"], dz2)
    dz_r = switch_cols_to_rows(comm, dz2.view(R, Rl, Hz))             # inverse of step 7
    dz2, _ = B.attention_bwd(bp, sv["pair_row"], dz_r.reshape(Rl * R, Hz).contiguous())
    dz_c = switch_rows_to_cols(comm, dz2.view(Rl, R, Hz))             # inverse of step 6
    dz2 = B.triangle_bwd(bp, sv["tri_in"], dz_c.reshape(R * Rl, Hz).contiguous(), reduce_scatter=rs)
    dz_r = switch_cols_to_rows(comm, dz2.view(R, Rl, Hz))             # inverse of step 5
    dz2 = B.triangle_bwd(bp, sv["tri_out"], dz_r.reshape(Rl * R, Hz).contiguous(), reduce_scatter=rs)
    dm2 = B.opm_bwd(bp, sv["opm"], dz2, dm_r_ready().reshape(S * Rl, Hm).contiguous(), reduce_scatter=rs)
    dm2 = B.transition_bwd(bp, sv["msa_trans"], dm2)
    dm2, _ = B.attention_bwd(bp, sv["msa_col"], dm2)
    dm_s = switch_cols_to_rows(comm, dm2.view(S, Rl, Hm))             # inverse of step 2
    dm2, dbias = B.attention_bwd(bp, sv["msa_row"], dm_s.reshape(Sl * R, Hm).contiguous())
    if N > 1:
        dbias = comm.reduce_scatter(dbias.view(nh, N, Rl, R).permute(1, 0, 2, 3))
    dz2 = B.msa_row_bias_bwd(bp, sv["bias"], dbias, dz2)
    B.SideStream.join()
    return dm2.view(Sl, R, Hm), dz2.view(Rl, R, Hz)


def shard_of(x, axis: int, comm: DapComm):
    """this rank's block of a full tensor (shard, sharding.py:114-123)."""
    n = comm.N
    if x.shape[axis] % n:
        raise ShardError(f"extent {x.shape[axis]} on axis {axis} not divisible by {n} devices")
    k = x.shape[axis] // n
    return x.narrow(axis, comm.rank * k, k).contiguous()


class DapStack:
    """N blocks under DAP on this rank (one process per GPU, NCCL).  Parameters are
    replicated; their gradients are summed over ranks with one all-reduce per block."""

    def __init__(self, cfg: EvoConfig, n_blocks: int, seed: int = 0, device="cuda", comm: DapComm | None = None,
                 params=None):
        from .config import init_block_params
        from .params import BlockLayout, BlockParams
        self.cfg = cfg
        self.comm = comm or DapComm()
        layout = BlockLayout(cfg)
        self.blocks = [BlockParams(params[i] if params is not None else init_block_params(cfg, seed + i), cfg,
                                   device=device, layout=layout) for i in range(n_blocks)]

    def shard_inputs(self, m, z, device):
        mt = torch.as_tensor(m).to(device=device, dtype=torch.bfloat16)
        zt = torch.as_tensor(z).to(device=device, dtype=torch.bfloat16)
        return shard_of(mt, 0, self.comm), shard_of(zt, 0, self.comm)

    def zero_grad(self):
        for b in self.blocks:
            b.zero_grad()

    def forward(self, m, z, save=True):
        saved = []
        for b in self.blocks:
            m, z, s = dap_block_fwd(b, self.comm, m, z, save)
            saved.append(s)
        return m, z, saved

    def backward(self, saved, dm, dz):
        # one gradient all-reduce per block (a 6.8 MB bucket at the training shape), issued async
        # as soon as the block's parameter gradients are final: it runs on the communicator's
        # stream under the previous block's backward; all are waited for before returning
        pending = []
        for b, s in zip(reversed(self.blocks), reversed(saved)):
            dm, dz = dap_block_bwd(b, self.comm, s, dm, dz)
            pending.append(self.comm.all_reduce_(b.grad, async_op=True))
        for w in pending:
            w.wait()
        return dm, dz

    def forward_backward(self, m, z, gm, gz):
        mo, zo, saved = self.forward(m, z, save=True)
        loss = (mo.float() * gm.float()).sum() + (zo.float() * gz.float()).sum()
        dm, dz = self.backward(saved, gm.to(torch.bfloat16).contiguous(), gz.to(torch.bfloat16).contiguous())
        return loss, dm, dz

    def e2e(self, m64, z64, gm64, gz64, steps, nb):
        """end-to-end timing through the API: each rank copies its shards from pinned host
        memory every step and reads the loss back."""
        dev = torch.device("cuda", torch.cuda.current_device())
        hs = [torch.tensor(a, dtype=torch.float32) for a in (m64, z64, gm64, gz64)]
        hs = [shard_of(h, 0, self.comm).pin_memory() for h in hs]
        hloss = torch.empty(1, dtype=torch.float32).pin_memory()
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(steps):
            m, z, gm, gz = (h.to(dev, non_blocking=True).bfloat16() for h in hs)
            self.zero_grad()
            loss, _, _ = self.forward_backward(m, z, gm, gz)
            hloss.copy_(loss.view(1), non_blocking=True)
            st.synchronize()
        b.record(st)
        torch.cuda.synchronize()
        ms = self.comm.all_reduce_max(a.elapsed_time(b) / steps)
        return {"value": round(ms / nb, 4), "unit": "ms/block", "h2d_bytes_per_step": sum(h.numel() * 4 for h in hs),
                "d2h_bytes_per_step": 4, "ms_per_step": round(ms, 3),
                "path": "DapStack.forward_backward per rank, pinned fp32 host shards in, loss read back"}


# ----------------------------------------------------------------------------- reference API
def dap_evoformer_block(m, z, p, cfg: EvoConfig, mesh: DeviceMesh, ledger: CommLedger | None = None):
    """dap_block.py:46-152: one block sharded over ``mesh``; full (m, z) in, full (m', z') out.

    * torch.distributed initialised with world size == mesh.n_devices: this process is
      rank `dist.get_rank()` (NCCL); outputs are all-gathered so every rank returns the
      full arrays, as the reference does.
    * otherwise: the mesh's ranks run as threads of this process on the current GPU
      (the reference's single-process simulation, with real kernels and collectives
      emulated by rendezvous).
    Inputs numpy (float64 in/out, like the reference) or torch CUDA tensors.
    """
    import numpy as np
    import torch.distributed as dist

    from .evoformer import _block_params, _check_msa, _check_pair, _to_dev
    _check_msa(m, cfg)
    _check_pair(z, cfg)
    n = mesh.n_devices
    if cfg.n_seq % n or cfg.n_res % n:
        raise ShardError(f"n_seq={cfg.n_seq} / n_res={cfg.n_res} not divisible by {n} devices")
    was_np = isinstance(m, np.ndarray)
    mt, _ = _to_dev(m)
    zt, _ = _to_dev(z)
    bp = _block_params(p, cfg)
    out = lambda t: t.double().cpu().numpy() if was_np else t
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == n:
        comm = DapComm(ledger=ledger)
        mo, zo, _ = dap_block_fwd(bp, comm, shard_of(mt, 0, comm), shard_of(zt, 0, comm), save=False)
        comm.ledger = None   # unsharding the result is not part of the block's traffic
        mf = comm.all_gather(mo).reshape(cfg.n_seq, cfg.n_res, cfg.h_msa)
        zf = comm.all_gather(zo).reshape(cfg.n_res, cfg.n_res, cfg.h_pair)
        comm.ledger = ledger
        return out(mf), out(zf)
    import threading
    tm = ThreadMesh(n)
    results: list = [None] * n
    errors: list = []
    dev = torch.cuda.current_device()

    def run(rank):
        try:
            torch.cuda.set_device(dev)
            comm = ThreadComm(tm, rank, ledger)
            results[rank] = dap_block_fwd(bp, comm, shard_of(mt, 0, comm), shard_of(zt, 0, comm), save=False)[:2]
        except BaseException as exc:  # noqa: BLE001 - re-raised in the caller
            errors.append(exc)
            tm.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in mesh.device_order]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    torch.cuda.synchronize()
    mf = torch.cat([r[0] for r in results], 0)
    zf = torch.cat([r[1] for r in results], 0)
    return out(mf), out(zf)
