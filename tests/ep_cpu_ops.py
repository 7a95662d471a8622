"""CPU reference ops for the EP tests (test infrastructure).

Implements the ExpertParallelSmoeMlp ``ops`` interface with torch indexing
and the NumPy oracle, so the multi-process communication and index algebra
of paper_2403_08245_b200.ep can be exercised with the gloo backend on CPU.
"""
import numpy as np
import torch

from oracle import scattermlp_oracle as orc
from paper_2403_08245_b200.router import GroupedOrder


def _np(t):
    return t.detach().cpu().numpy()


class CpuOps:
    @staticmethod
    def order(routing, num_experts):
        o, off = orc.compute_grouped_order(_np(routing.expert_idx), num_experts)
        return GroupedOrder(o=torch.from_numpy(o).to(torch.int32), bin_offsets=torch.from_numpy(off).to(torch.int32),
                            validate=False)

    @staticmethod
    def group(x, order_o32, fan_out, weights=None):
        w = None if weights is None else _np(weights)
        return torch.from_numpy(orc.group(_np(x), _np(order_o32).astype(np.int64), w, fan_out))

    @staticmethod
    def combine(p, y_hat):
        return torch.from_numpy(orc.combine(_np(p), _np(y_hat)))

    @staticmethod
    def combine_grad_p(dy, y_hat, s, j):
        return torch.from_numpy(orc.combine_grad_p(_np(dy), _np(y_hat), s, j))

    @staticmethod
    def fanout_reduce(g, fan_out):
        return torch.from_numpy(orc.fanout_reduce(_np(g), fan_out))

    @staticmethod
    def local_forward(r, w1, w2, o_loc, off_loc, activation):
        o, off = _np(o_loc).astype(np.int64), _np(off_loc).astype(np.int64)
        h_pre = orc.scatter2scatter(_np(r), _np(w1), o, off, 1, False, True)
        h = orc.act(h_pre, activation)
        y = orc.scatter2scatter(h, _np(w2), o, off, 1, True, False)
        return torch.from_numpy(y), (o, off, h_pre, h)

    @staticmethod
    def local_backward(r, w1, w2, saved, dy, activation):
        o, off, h_pre, h = saved
        gdy = orc.group(_np(dy), o)
        dw2 = orc.group_xty(h, gdy, off)
        dh = (orc.scatter2scatter(gdy, _np(w2), o, off, 1, True, True, transpose_w=True)
              * orc.act_grad(h_pre, activation)).astype(np.float32)
        xbar = orc.group(_np(r), o)
        dw1 = orc.group_xty(xbar, dh, off)
        dr = orc.scatter2scatter(dh, _np(w1), o, off, 1, True, False, transpose_w=True)
        return torch.from_numpy(dr), torch.from_numpy(dw1), torch.from_numpy(dw2)
