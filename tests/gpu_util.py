"""Helpers for the GPU parity tests (imported only by tests marked gpu)."""
import numpy as np
import torch

import paper_2403_08245_b200 as sm

DEV = "cuda"


def t(a, dtype=None):
    x = torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    return x.to(dtype) if dtype is not None else x


def order_of(idx, e):
    routing_idx = t(np.asarray(idx, dtype=np.int64))
    o, sorted_ids, offsets, inv = sm.router._sort_ids(routing_idx.reshape(-1), int(e))
    return sm.GroupedOrder(o=o, bin_offsets=offsets, sorted_expert_idxs=sorted_ids, inv=inv, validate=False)


def routing_of(idx, p, e):
    idx_t = t(np.asarray(idx, dtype=np.int64))
    p_t = t(np.asarray(p, dtype=np.float32))
    gate = torch.zeros((idx_t.shape[0], e), dtype=torch.float32, device=DEV).scatter_(1, idx_t, p_t)
    return sm.RoutingResult(expert_idx=idx_t, p=p_t, gate_full=gate, renormalized=False, validate=False)


def rel_err(got, want):
    g = got.detach().float().cpu().numpy().astype(np.float64) if torch.is_tensor(got) else np.asarray(got, np.float64)
    w = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(w)
    return float(np.linalg.norm(g - w) / (den if den > 0 else 1.0))


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def np_of(x):
    return x.detach().float().cpu().numpy()
