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
