"""Device-buffer management around the C ABI (torch is the allocator and stream source).

``CpmmEngine`` owns the caller-side buffers the ABI asks for (ctpt_query_sizes) and
drives the three calls of the hot path: format layout, plaintext precompute and
ctpt_matmul.  All arithmetic happens in libctpt.so.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import ctpt

# the largest d3_loc the limbs-in-TMEM skinny kernel (which forms the unsigned-U row sums itself)
# takes under CTPT_KERNEL_AUTO (ctpt.cu kFusedMaxD3)
TMEM_MAX_D3 = 256


def _u32_to_dev(a: np.ndarray, device) -> torch.Tensor:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).to(device, non_blocking=False)


def dev_to_u32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


class CpmmEngine:
    def __init__(self, spec: ctpt.Spec, device: str | torch.device = "cuda", alloc_ws: bool = True):
        """alloc_ws=False: the caller provides self.ws (e.g. one workspace shared by several engines
        whose problems run one after another)."""
        self.device = torch.device(device)
        self.spec = dataclasses.replace(spec)
        self.sizes = ctpt.query_sizes(self.spec)
        self.ws = (torch.empty(self.sizes.workspace_bytes, dtype=torch.uint8, device=self.device) if alloc_ws
                   else torch.empty(0, dtype=torch.uint8, device=self.device))
        self.ctmat = None
        self.plain = None

    # -- a1: format layout ----------------------------------------------------------------
    def layout(self, a_polys, b_polys, validate: bool = False) -> torch.Tensor:
        if self.sizes.rows_A == 0:  # structured-A: the a-polynomials are not read (Ã passes through)
            a = None
        else:
            a = a_polys if isinstance(a_polys, torch.Tensor) else _u32_to_dev(a_polys, self.device)
        b = b_polys if isinstance(b_polys, torch.Tensor) else _u32_to_dev(b_polys, self.device)
        if self.ctmat is None:
            self.ctmat = torch.empty(self.sizes.ctmat_bytes, dtype=torch.uint8, device=self.device)
        ctpt.layout(self.spec, a, b, self.ctmat, validate=validate)
        return self.ctmat

    # -- a2: plaintext precompute ------------------------------------------------------------
    def precompute(self, U, unsigned: str = "auto") -> int:
        """U's digit planes.  unsigned="auto" stores one u8 plane U + u_offset (lower tensor-core
        switching power under the 1000 W cap than sign-extended s8 digits: +5 % on the GEMM, +2–10 %
        in the power-bound skinny regime, profiles/r01/power_operands_c3gemm.jsonl,
        profiles/r02/u8_skinny_probe/) when U spans ≤ 255 values and the kernel ctpt_matmul will pick
        can correct for u_offset: k_gemm_tc (d3_loc > 256) and the limbs-in-TMEM skinny kernel
        (d3_loc ≤ TMEM_MAX_D3, which forms the row sums itself) — not the raw-byte kernel (d3_loc ≤ 32
        with fewer 64-row tiles than SMs).  "never" forces balanced s8 digits; "always" requires the
        u8 plane."""
        Ud = U if isinstance(U, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(U, dtype=np.int64))
        Ud = Ud.to(self.device)
        self.spec.kU = 4  # size the buffer for the worst case first
        self.spec.u_unsigned, self.spec.u_offset = 0, 0
        sz = ctpt.query_sizes(self.spec)
        self.plain = torch.empty(sz.plain_bytes, dtype=torch.uint8, device=self.device)
        self.spec.plain_per_prime = 0
        d3l = self.sizes.d3_loc
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        u8_kernel = d3l > 256 or (d3l <= TMEM_MAX_D3 and not (d3l <= 32 and (self.sizes.R + 63) // 64 < sms))
        want_u8 = unsigned == "always" or (unsigned == "auto" and u8_kernel and self.spec.d2 <= 33025)
        if want_u8:
            self.spec.kU = 1
            try:
                off = ctpt.plain_precompute_unsigned(self.spec, Ud, self.plain)
                self.spec.u_unsigned, self.spec.u_offset = 1, off
                self._resize_ws()
                return 1
            except ctpt.CtptError:
                if unsigned == "always":
                    raise
                self.spec.kU = 4
        kU = ctpt.plain_precompute(self.spec, Ud, self.plain)
        self.spec.kU = kU
        self._resize_ws()
        return kU

    def _resize_ws(self):
        """The workspace depends on the plane mode (row sums) — re-query once the mode is known."""
        self.sizes = ctpt.query_sizes(self.spec)
        if self.ws.numel() < self.sizes.workspace_bytes:
            self.ws = torch.empty(self.sizes.workspace_bytes, dtype=torch.uint8, device=self.device)

    def precompute_rns(self, Ures) -> int:
        Ud = Ures if isinstance(Ures, torch.Tensor) else _u32_to_dev(Ures, self.device)
        self.plain = torch.empty(self.sizes.plain_rns_bytes, dtype=torch.uint8, device=self.device)
        self.spec.u_unsigned, self.spec.u_offset = 0, 0
        kU = ctpt.plain_precompute_rns(self.spec, Ud, self.plain)
        self.spec.kU = kU
        self.spec.plain_per_prime = 1
        self._resize_ws()
        return kU

    # -- a3–a6: the hot path -------------------------------------------------------------------
    def alloc_outputs(self):
        AU = torch.empty(max(1, self.sizes.out_AU_bytes // 4), dtype=torch.int32, device=self.device)
        BU = torch.empty(self.sizes.out_BU_bytes // 4, dtype=torch.int32, device=self.device)
        return AU, BU

    def matmul(self, AU=None, BU=None, stream=None):
        if AU is None:
            AU, BU = self.alloc_outputs()
        ctpt.matmul(self.spec, self.ctmat, self.plain, AU, BU, self.ws, stream=stream)
        return AU, BU

    def outputs_numpy(self, AU: torch.Tensor, BU: torch.Tensor):
        L = len(self.spec.primes) - self.spec.rescale  # Rescale drops the last prime
        d3l = self.sizes.d3_loc
        ra = self.sizes.rows_A
        AUn = dev_to_u32(AU)[:L * d3l * ra].reshape(L, d3l, ra)
        return AUn, dev_to_u32(BU).reshape(L, d3l, self.spec.d1)
