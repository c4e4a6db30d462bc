"""GCN neighbour aggregation on top of DA-SpMM (BASELINE configs[2]: the
Reddit-scale aggregation is exactly C = Â · H with N = 128 feature columns).

A GCN layer (Kipf & Welling) computes H' = act(Â · H · W + b) with the normalised
adjacency Â = D^-1/2 (A + I) D^-1/2. The sparse product runs through the device-resident
DA-SpMM path (selector + chosen kernel on the GPU, `spmm_selected`); the dense transform
H · W is a plain cuBLAS GEMM. The transform is applied first when it narrows the
features (out < in), so the SpMM runs on the narrower operand.

Graph preprocessing (self loops, degrees, the symmetric scaling of the values) is a
one-time device pass with torch ops; the handle then stays resident across layers and
epochs.
"""
from __future__ import annotations

import os

import torch

from . import spmmkit as sk


def normalized_adjacency(num_nodes: int, row_offsets: torch.Tensor, col_indices: torch.Tensor,
                         values: torch.Tensor | None = None, add_self_loops: bool = True):
    """Â = D^-1/2 (A + I) D^-1/2 as device CSR (int32 offsets/cols, fp32 values).
    Existing diagonal entries are kept (and I added on top, as in the GCN definition)."""
    dev = row_offsets.device
    rp = row_offsets.to(torch.int64)
    ci = col_indices.to(torch.int64)
    va = values.to(torch.float32) if values is not None else torch.ones(ci.numel(), device=dev)
    rows = torch.repeat_interleave(torch.arange(num_nodes, device=dev), rp[1:] - rp[:-1])
    if add_self_loops:
        eye = torch.arange(num_nodes, device=dev)
        rows = torch.cat([rows, eye])
        ci = torch.cat([ci, eye])
        va = torch.cat([va, torch.ones(num_nodes, device=dev)])
        order = torch.argsort(rows * num_nodes + ci)
        rows, ci, va = rows[order], ci[order], va[order]
    deg = torch.zeros(num_nodes, device=dev).index_add_(0, rows, va)
    dinv = torch.where(deg > 0, deg.rsqrt(), torch.zeros_like(deg))
    va = dinv[rows] * va * dinv[ci]
    counts = torch.bincount(rows, minlength=num_nodes)
    rp_out = torch.zeros(num_nodes + 1, dtype=torch.int64, device=dev)
    rp_out[1:] = torch.cumsum(counts, 0)
    return rp_out.to(torch.int32), ci.to(torch.int32), va.contiguous()


class GCNGraph:
    """A graph's normalised adjacency, resident on the device as a DA-SpMM handle."""

    def __init__(self, num_nodes: int, row_offsets, col_indices, values=None,
                 add_self_loops: bool = True, model_path: str | None = None):
        rp, ci, va = normalized_adjacency(num_nodes, row_offsets, col_indices, values,
                                          add_self_loops)
        self.num_nodes = num_nodes
        self._arrays = (rp, ci, va)  # the handle borrows them
        self.adj = sk.DeviceCsr.from_device(num_nodes, num_nodes, rp, ci, va)
        path = model_path or os.path.join(os.path.dirname(__file__), "models",
                                          "b200_selector.txt")
        self.model = sk.load_selector(open(path).read())
        self._out = {}  # (N, dtype) -> the graph's own output buffer

    def aggregate(self, H: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Â · H (row-major fp32, N = H.shape[1] columns) through DA-SpMM.

        Without ``out`` the result lands in a buffer the graph owns (one per width and
        dtype), which the next aggregate of the same width overwrites — clone it to keep
        it. Layer after layer thus allocates nothing on the SpMM side."""
        H = H.contiguous()
        if out is None:
            key = (H.shape[1], H.dtype)
            out = self._out.get(key)
            if out is None or out.device != H.device:
                out = torch.empty(self.num_nodes, H.shape[1], device=H.device, dtype=H.dtype)
                self._out[key] = out
        sk.spmm_selected(self.adj, self.model, H, out)
        return out


class GCNLayer(torch.nn.Module):
    """H' = act(Â · H · W + b); forward only (inference / feature propagation)."""

    def __init__(self, in_features: int, out_features: int, bias: bool = True,
                 activation=torch.relu):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.empty(in_features, out_features))
        self.bias = torch.nn.Parameter(torch.zeros(out_features)) if bias else None
        self.activation = activation
        torch.nn.init.xavier_uniform_(self.weight)

    @torch.no_grad()
    def forward(self, graph: GCNGraph, H: torch.Tensor) -> torch.Tensor:
        W = self.weight
        if W.shape[1] < W.shape[0]:  # transform first: the SpMM runs on fewer columns
            Z = graph.aggregate(H @ W)
        else:
            Z = graph.aggregate(H) @ W
        if self.bias is not None:
            Z = Z + self.bias
        return self.activation(Z) if self.activation is not None else Z


__all__ = ["normalized_adjacency", "GCNGraph", "GCNLayer"]
