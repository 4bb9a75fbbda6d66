"""Multi-GPU host logic (one process per GPU, torch.distributed over NCCL/NVLink).

Two partitions of the decode-attention work:
  * batch x KV-head sharding (large batch, BASELINE configs[2]): units are independent, each rank
    owns a contiguous slice of sequences -> no collective on the data path ("scaling": weak).
  * sequence sharding (single 196k-token sequence, configs[3]): rank r attends tokens
    [r*N/P, (r+1)*N/P) through vecinfer_attn_decode's tok_begin/tok_end hook, producing a
    normalised partial (o_r, L_r) of 32 x (128 + 1) fp32 per sequence; ONE all-gather exchanges
    the P partials and every rank merges them with vecinfer_merge_lse in rank order, so all
    ranks hold bitwise-identical outputs.
The functions here only compute ranges and move partials; the arithmetic is in the kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_tokens: int, rank: int, world: int, align: int = 32) -> tuple[int, int]:
    """Contiguous token shard of rank `rank`: boundaries rounded to `align` tokens, union = [0, n)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = -(-n_tokens // world)
    per = -(-per // align) * align
    b = min(rank * per, n_tokens)
    e = min(b + per, n_tokens)
    return b, e


def batch_shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice of sequences owned by `rank` (batch x KV-head sharding)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = -(-batch // world)
    b = min(rank * per, batch)
    return b, min(b + per, batch)


def gather_partials(o_local: torch.Tensor, lse_local: torch.Tensor, group=None):
    """All-gather the per-rank partials into [P, ...] tensors in rank order (one collective each
    for o and lse; 16.1 KiB + 128 B per rank for B = 1, H_q = 32)."""
    world = dist.get_world_size(group)
    o_all = torch.empty((world,) + tuple(o_local.shape), dtype=o_local.dtype, device=o_local.device)
    l_all = torch.empty((world,) + tuple(lse_local.shape), dtype=lse_local.dtype, device=lse_local.device)
    if o_local.is_cuda:
        dist.all_gather_into_tensor(o_all, o_local.contiguous(), group=group)
        dist.all_gather_into_tensor(l_all, lse_local.contiguous(), group=group)
    else:   # gloo path (host-side tests)
        dist.all_gather(list(o_all.unbind(0)), o_local.contiguous(), group=group)
        dist.all_gather(list(l_all.unbind(0)), lse_local.contiguous(), group=group)
    return o_all, l_all


def gather_partials_packed(o_local: torch.Tensor, lse_local: torch.Tensor, group=None):
    """Same exchange with ONE collective: lse is packed behind o in a single fp32 buffer."""
    world = dist.get_world_size(group)
    flat = torch.cat([o_local.reshape(-1).float(), lse_local.reshape(-1).float()])
    out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    if flat.is_cuda:
        dist.all_gather_into_tensor(out, flat, group=group)
    else:
        dist.all_gather(list(out.view(world, -1).unbind(0)), flat, group=group)
    out = out.view(world, -1)
    no = o_local.numel()
    return (out[:, :no].reshape((world,) + tuple(o_local.shape)),
            out[:, no:].reshape((world,) + tuple(lse_local.shape)).contiguous())


class P2PExchange:
    """Fused cross-GPU exchange + LSE merge over peer memory (vecinfer_merge_lse_p2p): the
    replacement for gather_partials_packed + vecinfer_merge_lse on the sequence-sharded path.

    Setup (collective over `group`, any backend that can all_gather_object): every rank creates its
    window (library cudaMalloc) and exports a CUDA IPC handle; the handles are all-gathered and the
    peers' windows mapped.  merge() then runs ONE kernel per call: remote stores of this rank's
    partial rows into every window, per-row release flags, acquire-polling of the own window, and
    the rank-order merge.  Ranks must call merge() the same number of times with the same shapes.
    """

    def __init__(self, rows_max: int, D: int, device: torch.device, group=None):
        import ctypes

        from . import _lib
        self._lib = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows_max, self.D, self.device = rows_max, D, device
        nbytes = self._lib.vecinfer_p2p_window_bytes(self.world, rows_max, D)
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        with torch.cuda.device(device):
            _lib.check("vecinfer_p2p_window_create",
                       self._lib.vecinfer_p2p_window_create(nbytes, ctypes.addressof(own), ctypes.addressof(handle)))
        self._own = own.value
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        ptrs = []
        self._opened = []
        with torch.cuda.device(device):
            for p, h in enumerate(handles):
                if p == self.rank:
                    ptrs.append(self._own)
                    continue
                w = ctypes.c_void_p()
                hb = (ctypes.c_char * 64).from_buffer_copy(h)
                _lib.check("vecinfer_p2p_window_open",
                           self._lib.vecinfer_p2p_window_open(ctypes.addressof(hb), ctypes.addressof(w)))
                ptrs.append(w.value)
                self._opened.append(w.value)
        self.windows = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self.epoch = 0
        self._group = group

    def merge(self, o_local: torch.Tensor, lse_local: torch.Tensor, out: torch.Tensor | None = None,
              lse: torch.Tensor | None = None, o_dtype: torch.dtype = torch.float32):
        """o_local fp32 [B, H_q, D], lse_local fp32 [B, H_q] -> merged (o, lse) on every rank."""
        import ctypes

        from . import _lib
        B, Hq, D = o_local.shape
        if B * Hq > self.rows_max or D != self.D:
            raise ValueError("partials larger than the window")
        if not (o_local.is_contiguous() and lse_local.is_contiguous()):
            raise ValueError("partials must be contiguous")
        if out is None:
            out = torch.empty(B, Hq, D, dtype=o_dtype, device=o_local.device)
        if lse is None:
            lse = torch.empty(B, Hq, dtype=torch.float32, device=o_local.device)
        self.epoch += 1   # calls made (the kernel keeps the exchange epoch on the device: graph-safe)
        stream = ctypes.c_void_p(torch.cuda.current_stream(o_local.device).cuda_stream)
        _lib.check("vecinfer_merge_lse_p2p", self._lib.vecinfer_merge_lse_p2p(
            ctypes.c_void_p(o_local.data_ptr()), ctypes.c_void_p(lse_local.data_ptr()),
            ctypes.c_void_p(self.windows.data_ptr()), self.world, self.rank, B, Hq, D, 0,
            ctypes.c_void_p(out.data_ptr()), 1 if out.dtype == torch.float32 else 0, ctypes.c_void_p(lse.data_ptr()),
            ctypes.c_void_p(self.err.data_ptr()), stream))
        return out, lse

    def close(self):
        """Unmap the peers' windows and free the own one (collective: call on every rank)."""
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self._group)
        for w in self._opened:
            self._lib.vecinfer_p2p_window_close(w)
        self._opened = []
        dist.barrier(group=self._group)
        if self._own:
            self._lib.vecinfer_p2p_window_destroy(self._own)
            self._own = None


class XRankWindows:
    """Peer-memory windows of the cross-GPU merge fused INTO the attention launch
    (vecinfer_attn_decode_xr / vecinfer_decode_step_xr; "N4's epilogue stores partials
    straight into peers' symmetric windows").  Pass as `xr=` to vecinfer.attn_decode / decode_step:
    each rank attends its own sequence shard and the launch returns the merged o, lse on every rank.

    Setup is collective over `group` (CUDA IPC handles all-gathered, peers mapped), as P2PExchange.
    XRankWindows.local(P, ...) builds P descriptors over P windows of ONE process (ranks run as
    concurrent launches on P streams of one GPU: the single-GPU functional tests)."""

    def __init__(self, rows_max: int, D: int, device: torch.device, group=None, _local=None):
        import ctypes

        from . import _lib
        self._lib = _lib.load()
        self.rows_max, self.D, self.device = rows_max, D, device
        self._opened, self._own, self._group = [], None, group
        if _local is not None:   # (world, rank, windows tensor, err tensor, keep-alive buffers)
            self.world, self.rank, self.windows, self.err, self._bufs = _local
        else:
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
            nbytes = self._lib.vecinfer_xr_window_bytes(self.world, rows_max, D)
            own = ctypes.c_void_p()
            handle = (ctypes.c_char * 64)()
            with torch.cuda.device(device):
                _lib.check("vecinfer_p2p_window_create",
                           self._lib.vecinfer_p2p_window_create(nbytes, ctypes.addressof(own), ctypes.addressof(handle)))
            self._own = own.value
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(handle), group=group)
            ptrs = []
            with torch.cuda.device(device):
                for p, h in enumerate(handles):
                    if p == self.rank:
                        ptrs.append(self._own)
                        continue
                    w = ctypes.c_void_p()
                    hb = (ctypes.c_char * 64).from_buffer_copy(h)
                    _lib.check("vecinfer_p2p_window_open",
                               self._lib.vecinfer_p2p_window_open(ctypes.addressof(hb), ctypes.addressof(w)))
                    ptrs.append(w.value)
                    self._opened.append(w.value)
            self.windows = torch.tensor(ptrs, dtype=torch.int64, device=device)
            self.err = torch.zeros(1, dtype=torch.int32, device=device)
            self._bufs = []
        self._struct = _lib.XRank(self.world, self.rank, self.windows.data_ptr(), rows_max, self.err.data_ptr())
        self.desc = ctypes.pointer(self._struct)

    @classmethod
    def local(cls, P: int, rows_max: int, D: int, device: torch.device):
        """P single-process ranks over P in-process windows (one per rank, zero-filled)."""
        from . import _lib
        nbytes = _lib.load().vecinfer_xr_window_bytes(P, rows_max, D)
        bufs = [torch.zeros(nbytes, dtype=torch.uint8, device=device) for _ in range(P)]
        windows = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=device)
        err = torch.zeros(1, dtype=torch.int32, device=device)
        return [cls(rows_max, D, device, _local=(P, r, windows, err, bufs)) for r in range(P)]

    def close(self):
        """Unmap the peers' windows and free the own one (collective unless built by local())."""
        if self._own is None:
            return
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self._group)
        for w in self._opened:
            self._lib.vecinfer_p2p_window_close(w)
        self._opened = []
        dist.barrier(group=self._group)
        self._lib.vecinfer_p2p_window_destroy(self._own)
        self._own = None


class SeqShardedStep:
    """One decode step of an L-layer model whose single long sequence is sharded over the ranks
    (BASELINE configs[3]): for every layer, this rank's attention over its token
    shard [tok_begin, tok_end) writes a normalised partial (o_r, L_r), and that layer's partials are
    exchanged and LSE-merged BEFORE the next layer runs -- the next layer's query depends on this
    layer's output in a real model, so the exchange is paid once per layer, not once per step.

    exchange="xr": the merge fused INTO the attention launch (XRankWindows; graph-safe, no exchange launch).
    exchange="p2p": the fused peer-memory kernel (P2PExchange, one launch per layer; graph-safe).
    exchange="allgather": one packed all-gather per layer + vecinfer_merge_lse (NCCL on device
    tensors; gloo through host copies for the single-GPU functional tests).
    Outputs: self.o [L, B, H_q, D] (o_dtype), self.lse [L, B, H_q], identical on every rank.
    """

    def __init__(self, layers: int, B: int, H_q: int, D: int, n_tokens: int, device: torch.device,
                 H_kv: int = 8, exchange: str = "p2p", o_dtype: torch.dtype = torch.float32, group=None):
        from . import vecinfer as vi
        if exchange not in ("xr", "p2p", "allgather"):
            raise ValueError("exchange must be 'xr', 'p2p' or 'allgather'")
        self.vi = vi
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.L, self.B, self.H_q, self.D = layers, B, H_q, D
        self.tok_begin, self.tok_end = shard_range(n_tokens, self.rank, self.world)
        n_local = self.tok_end - self.tok_begin
        self.o_part = torch.empty(layers, B, H_q, D, dtype=torch.float32, device=device)
        self.lse_part = torch.empty(layers, B, H_q, dtype=torch.float32, device=device)
        self.o = torch.empty(layers, B, H_q, D, dtype=o_dtype, device=device)
        self.lse = torch.empty(layers, B, H_q, dtype=torch.float32, device=device)
        self.workspace = [vi.attn_workspace(B, H_q, H_kv, max(n_local, 1), device=device) for _ in range(layers)]
        self.exchange = exchange
        self.p2p = P2PExchange(B * H_q, D, device, group=group) if exchange == "p2p" else None
        self.xr = XRankWindows(B * H_q, D, device, group=group) if exchange == "xr" else None
        self.device = device

    def exchange_layer(self, l: int):
        """Exchange + merge layer l's partials (every rank ends with the same o[l], lse[l])."""
        if self.p2p is not None:
            self.p2p.merge(self.o_part[l], self.lse_part[l], out=self.o[l], lse=self.lse[l])
            return
        o_p, l_p = self.o_part[l], self.lse_part[l]
        host = dist.get_backend(self.group) == "gloo"
        o_g, l_g = gather_partials_packed(o_p.cpu() if host else o_p, l_p.cpu() if host else l_p, group=self.group)
        if host:
            o_g, l_g = o_g.to(self.device), l_g.to(self.device)
        self.vi.merge_lse(o_g.contiguous(), l_g.contiguous(), o_dtype=self.o.dtype, out=self.o[l], lse=self.lse[l])

    def run(self, attend):
        """attend(l, o_part_l, lse_part_l) launches layer l's shard attention (e.g. vi.attn_decode with
        tok_begin/tok_end and out=/lse=); the exchange of layer l follows it immediately.
        exchange="xr": attend(l, o_l, lse_l, xr=windows) must pass xr= to vi.attn_decode / decode_step,
        which then writes the MERGED layer output itself (one launch per layer, no exchange)."""
        for l in range(self.L):
            if self.xr is not None:
                attend(l, self.o[l], self.lse[l], xr=self.xr)
                continue
            attend(l, self.o_part[l], self.lse_part[l])
            self.exchange_layer(l)

    def error(self) -> int:
        """Non-zero if a peer partial timed out in the fused exchange (VECINFER_FLAG_P2P_TIMEOUT)."""
        if self.xr is not None:
            return int(self.xr.err.item())
        return int(self.p2p.err.item()) if self.p2p is not None else 0

    def close(self):
        if self.p2p is not None:
            self.p2p.close()
            self.p2p = None
        if self.xr is not None:
            self.xr.close()
            self.xr = None
