"""VQ KV cache with a full-precision residual window for one attention layer (plumbing only).

Protocol ("the residual length for all methods is set to 128"; SPEC S:228-229 flush policy):
the newest tokens of each sequence stay as raw bf16 k, v rows; when an append brings the window to
2R rows, the oldest R are encoded into the VQ cache in one bulk vecinfer_encode_kv call (Eq. 8/9)
and the window shifts down BEFORE that step attends, so attention never sees more than 2R - 1
window rows.  The flush of the oldest R rows does not involve the new token, so it is issued
before the step's single vecinfer_decode_step launch, which copies the new token into the window
and attends codes + window.  Deviation (R22): the window keeps RAW keys and the kernel
scores them with the raw query (q k^T = q~ k~^T exactly in real arithmetic, Eq. 7), where SPEC
S:250 stores them already transformed; the codes of flushed rows are identical either way (the
encoder transforms).  All arithmetic is in the CUDA kernels; this class only owns buffers and
lengths (uniform across the batch).
"""
from __future__ import annotations

import torch

from . import vecinfer as vi


class VQKVCache:
    def __init__(self, B: int, H_kv: int, n_cap: int, lam: torch.Tensor, inv_lambda: torch.Tensor,
                 ck: torch.Tensor, cv: torch.Tensor, residual: int = 128, kcfg=vi.B2D4, vcfg=vi.B2D4,
                 device="cuda", H_q: int | None = None):
        """H_q defaults to 4 * H_kv (Llama-3.1-8B grouping); the head dim D comes from kcfg."""
        self.B, self.H, self.R = B, H_kv, residual
        self.lam, self.inv, self.ck, self.cv = lam, inv_lambda, ck, cv
        self.kcfg, self.vcfg = kcfg, vcfg
        self.kc = torch.zeros(B, H_kv, n_cap, kcfg.row_bytes, dtype=torch.uint8, device=device)
        self.vc = torch.zeros(B, H_kv, n_cap, vcfg.row_bytes, dtype=torch.uint8, device=device)
        D = kcfg.head_dim
        self.H_q = H_q if H_q is not None else 4 * H_kv
        self.kr = torch.zeros(B, H_kv, 2 * residual, D, dtype=torch.bfloat16, device=device)
        self.vr = torch.zeros_like(self.kr)
        self.n_q = 0          # quantised tokens
        self.n_r = 0          # residual rows
        self.seq = torch.zeros(B, dtype=torch.int32, device=device)
        self.rlen = torch.zeros(B, dtype=torch.int32, device=device)
        self.ws = vi.decode_step_workspace(B, self.H_q, H_kv, n_cap, kcfg, vcfg, device=device)
        self.enc_ws = vi.encode_workspace(B, residual, H_kv, kcfg, vcfg, device=device)

    def _flush(self):
        """Encode the oldest R residual rows into the codes, shift the window down by R."""
        R = self.R
        k = self.kr[:, :, :R].permute(0, 2, 1, 3)        # [B, R, H, D] view (strided)
        v = self.vr[:, :, :R].permute(0, 2, 1, 3)
        wp = torch.full((self.B,), self.n_q, dtype=torch.int32, device=self.kc.device)
        vi.encode_kv(k, v, self.inv, self.ck, self.cv, self.kc, self.vc, wp, self.kcfg, self.vcfg,
                     workspace=self.enc_ws)
        self.kr[:, :, :R].copy_(self.kr[:, :, R:2 * R].clone())
        self.vr[:, :, :R].copy_(self.vr[:, :, R:2 * R].clone())
        self.n_q += R
        self.n_r -= R

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, out=None, lse=None):
        """One decode step: append (k_new, v_new) [B, H_kv, D] to the window and attend q [B, H_q, D]."""
        if q.shape[1] != self.H_q:
            raise ValueError(f"q has {q.shape[1]} heads, the cache was sized for H_q = {self.H_q}")
        if self.R > 0 and self.n_r == 2 * self.R - 1:   # this append fills the window: flush first
            self._flush()
        self.n_r += 1
        self.seq.fill_(self.n_q)
        self.rlen.fill_(self.n_r)
        return vi.decode_step(q, k_new, v_new, self.lam, self.inv, self.ck, self.cv, self.kc, self.vc, self.seq,
                              self.seq, kcfg=self.kcfg, vcfg=self.vcfg, out=out, lse=lse, workspace=self.ws,
                              k_res=self.kr, v_res=self.vr, res_lens=self.rlen, append_to_residual=True)


class PagedVQCache:
    """Ragged batch of sequences over one shared page pool (serving integration; SURVEY §8(f) NEXT-4,
    the paper's stated limitation P:679).  Plumbing only: a free-list page allocator, per-slot block
    tables and lengths; every byte of codes is written and read by the CUDA kernels
    (vecinfer_encode_kv_paged for prefill, vecinfer_decode_step_paged for each step).

    * K / V code pools [n_pages, H_kv, page_size, row] (page_size a power of two >= 32).
    * Slot s holds one sequence: block-table row s lists its pages in token order (-1 = none).
    * add(s, k, v): prefill T tokens (pages allocated for them), remove(s): pages back to the pool.
    * step(q, k_new, v_new, slots): one decode step of the given slots -- a page is allocated when a
      sequence crosses a page boundary, then one decode_step launch over the compact batch appends the
      new token at row len and attends [0, len + 1).
    """

    def __init__(self, max_seqs: int, H_kv: int, n_pages: int, page_size: int, max_len: int, lam: torch.Tensor,
                 inv_lambda: torch.Tensor, ck: torch.Tensor, cv: torch.Tensor, kcfg=vi.B2D4, vcfg=vi.B2D4,
                 H_q: int | None = None, device="cuda"):
        if page_size < 32 or page_size & (page_size - 1):
            raise ValueError("page_size must be a power of two >= 32")
        self.S, self.H, self.ps, self.device = max_seqs, H_kv, page_size, device
        self.H_q = H_q if H_q is not None else 4 * H_kv
        self.lam, self.inv, self.ck, self.cv, self.kcfg, self.vcfg = lam, inv_lambda, ck, cv, kcfg, vcfg
        self.pages_per_seq = -(-max_len // page_size)
        self.kpool = torch.zeros(n_pages, H_kv, page_size, kcfg.row_bytes, dtype=torch.uint8, device=device)
        self.vpool = torch.zeros(n_pages, H_kv, page_size, vcfg.row_bytes, dtype=torch.uint8, device=device)
        self.free = list(range(n_pages - 1, -1, -1))            # stack of free page ids
        self.bt_host = [[] for _ in range(max_seqs)]             # pages of each slot, in token order
        self.bt = torch.full((max_seqs, self.pages_per_seq), -1, dtype=torch.int32, device=device)
        self.lens = [0] * max_seqs
        self.ws = vi.decode_step_workspace(max_seqs, self.H_q, H_kv, self.pages_per_seq * page_size, kcfg, vcfg,
                                           device=device)

    @property
    def pages_in_use(self) -> int:
        return sum(len(p) for p in self.bt_host)

    def _grow(self, s: int, n_tokens: int):
        need = -(-n_tokens // self.ps)
        if need > self.pages_per_seq:
            raise ValueError(f"slot {s}: {n_tokens} tokens exceed max_len")
        while len(self.bt_host[s]) < need:
            if not self.free:
                raise RuntimeError("page pool exhausted")
            p = self.free.pop()
            self.bt[s, len(self.bt_host[s])] = p
            self.bt_host[s].append(p)

    def add(self, s: int, k: torch.Tensor, v: torch.Tensor):
        """Prefill slot s with k, v [T, H_kv, D] (bf16)."""
        if self.lens[s] or self.bt_host[s]:
            raise ValueError(f"slot {s} is in use")
        T = k.shape[0]
        self._grow(s, T)
        wp = torch.zeros(1, dtype=torch.int32, device=self.device)
        ws = vi.encode_workspace(1, T, self.H, self.kcfg, self.vcfg, device=self.device)
        vi.encode_kv(k[None], v[None], self.inv, self.ck, self.cv, self.kpool, self.vpool, wp, self.kcfg, self.vcfg,
                     workspace=ws, block_table=self.bt[s:s + 1])
        self.lens[s] = T

    def remove(self, s: int):
        """Release slot s and its pages."""
        self.free.extend(reversed(self.bt_host[s]))
        self.bt_host[s] = []
        self.bt[s].fill_(-1)
        self.lens[s] = 0

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, slots: list[int], out=None, lse=None):
        """q [n, H_q, D], k_new / v_new [n, H_kv, D] for the n given slots (in that order)."""
        for s in slots:
            self._grow(s, self.lens[s] + 1)
        idx = torch.tensor(slots, dtype=torch.long, device=self.device)
        wp = torch.tensor([self.lens[s] for s in slots], dtype=torch.int32, device=self.device)
        o, L = vi.decode_step(q, k_new, v_new, self.lam, self.inv, self.ck, self.cv, self.kpool, self.vpool, wp, wp + 1,
                              kcfg=self.kcfg, vcfg=self.vcfg, out=out, lse=lse, workspace=self.ws,
                              block_table=self.bt.index_select(0, idx).contiguous())
        for s in slots:
            self.lens[s] += 1
        return o, L
