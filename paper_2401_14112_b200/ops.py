"""torch custom op over the fused linear: `torch.ops.fpx.linear`.

    y = torch.ops.fpx.linear(x, streams_hi, streams_lo, scales, exp_bits, man_bits,
                             rows_p, cols_p, bias, activation)

x: [N, K] fp16 CUDA; streams / scales: the PackedWeights tensors; bias:
optional fp32 [rows_p]; activation: "none" | "relu" | "silu" | "gelu_tanh".
Returns fp16 [N, rows_p].  Registered with a fake (meta) implementation so
it traces under torch.compile / export without running the kernel; the CUDA
implementation is fpx_linear_ex through the C-ABI (no fallback).
`FpxLinear` wraps it as an nn.Module holding the packed weights in HBM.
"""
from __future__ import annotations

import torch

from . import fpx as F

_LIB = "fpx"


@torch.library.custom_op(f"{_LIB}::linear", mutates_args=())
def linear_op(x: torch.Tensor, stream_hi: torch.Tensor, stream_lo: torch.Tensor, scales: torch.Tensor,
              exp_bits: int, man_bits: int, rows_p: int, cols_p: int, orig_cols: int, bias: torch.Tensor | None,
              activation: str) -> torch.Tensor:
    fmt = F.FpxFormat(exp_bits, man_bits)
    p = F.PackedWeights(fmt, F.SplitScheme.for_format(fmt), rows_p, cols_p, rows_p, orig_cols,
                        [stream_hi, stream_lo], scales)
    return F.linear(x, p, bias=bias, activation=None if activation == "none" else activation,
                    out_dtype=torch.float16)


@linear_op.register_fake
def _(x, stream_hi, stream_lo, scales, exp_bits, man_bits, rows_p, cols_p, orig_cols, bias, activation):
    return x.new_empty((x.shape[0], rows_p), dtype=torch.float16)


class FpxLinear(torch.nn.Module):
    """nn.Linear replacement: weights quantised + pre-packed once, resident
    in HBM; forward(x [.., K] fp16) -> [.., out_features] fp16."""

    def __init__(self, weight: torch.Tensor, bias: torch.Tensor | None = None, fmt: F.FpxFormat | None = None,
                 activation: str = "none"):
        super().__init__()
        fmt = fmt or F.FpxFormat.e3m2()
        p = F.pack(F.quantize_matrix(weight.detach().float().cuda(), fmt))
        self.out_features, self.in_features = weight.shape
        self.fmt, self.rows_p, self.cols_p, self.orig_cols = fmt, p.rows, p.cols, p.orig_cols
        self.register_buffer("stream_hi", p.streams[0])
        self.register_buffer("stream_lo", p.streams[1])
        self.register_buffer("scales", p.scales)
        self.register_buffer("bias", None if bias is None else bias.detach().float().cuda())
        self.activation = activation

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        lead = x.shape[:-1]
        y = torch.ops.fpx.linear(x.reshape(-1, x.shape[-1]).half(), self.stream_hi, self.stream_lo, self.scales,
                                 self.fmt.exp_bits, self.fmt.man_bits, self.rows_p, self.cols_p, self.orig_cols,
                                 self.bias, self.activation)
        return y[:, :self.out_features].reshape(*lead, self.out_features)
