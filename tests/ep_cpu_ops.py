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
    def gather(x, rows_o32, fan_out):
        return torch.from_numpy(orc.group(_np(x), _np(rows_o32).astype(np.int64), None, fan_out))

    @staticmethod
    def fanout_reduce(g, fan_out):
        return torch.from_numpy(orc.fanout_reduce(_np(g), fan_out))

    @staticmethod
    def local_forward(r, p_recv, w1, w2, off_loc, activation, wait=None):
        """The scaled expert MLP (p moved through layer 2), f64 accumulate, f32 storage."""
        off = _np(off_loc).astype(np.int64)
        o = np.arange(r.shape[0], dtype=np.int64)
        h_pre = orc.scatter2scatter(_np(r), _np(w1), o, off, 1, True, True)
        hp = (_np(p_recv).astype(np.float64)[:, None] * orc.act(h_pre, activation).astype(np.float64)).astype(np.float32)
        y = orc.scatter2scatter(hp, _np(w2), o, off, 1, True, True)
        return torch.from_numpy(y), (o, off, h_pre, hp)

    @staticmethod
    def local_backward(r, p_recv, w1, w2, saved, dy, activation):
        o, off, h_pre, hp = saved
        p = _np(p_recv).astype(np.float64)[:, None]
        dyn = _np(dy)
        dw2 = orc.group_xty(hp, dyn, off)
        g = orc.scatter2scatter(dyn, _np(w2), o, off, 1, True, True, transpose_w=True).astype(np.float64)
        dp = (g * orc.act(h_pre, activation).astype(np.float64)).sum(1).astype(np.float32)
        dh = (p * g * orc.act_grad(h_pre, activation).astype(np.float64)).astype(np.float32)
        dw1 = orc.group_xty(_np(r), dh, off)
        dr = orc.scatter2scatter(dh, _np(w1), o, off, 1, True, True, transpose_w=True)
        return torch.from_numpy(dr), torch.from_numpy(dw1), torch.from_numpy(dw2), torch.from_numpy(dp)
