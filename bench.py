"""SMoE MLP fwd+bwd benchmark (BASELINE.json metric) — one JSON line on rank 0.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1|C2|C0] [--impl ours|reference]

A step = one pass of the ParallelLinear hot path over one batch: the routing
sort (flatten_and_sort), smoe_mlp_forward(training=True) and
smoe_mlp_backward, at the configuration BASELINE.json's metric is quoted on
(configs[1], "C1": Mixtral-8x7B MLP layer, T=32768, d_model=4096,
d_expert=14336, E=8, k=2, bf16).  Inputs are synthetic, weights random-init;
routing is a softmax gate + stable top-k computed once outside the timed
region (as the reference bench does, bench.py:120-130).

value  : tokens/s with inputs resident in HBM (device time, CUDA events).
e2e    : the same step through the public API from pinned HOST buffers:
         X, dY, expert ids and p copied H2D, dX and dp copied D2H, inside the
         timed region.
roofline: the dominant kernel (the GEMM with the largest share of the step,
         the grouped-K weight-gradient GEMM at C1/C2): its mean launch
         duration inside the timed steps (CUDA events around each launch on
         its stream, launch_timer.py); algorithmic FLOPs = 2*T*k*d*d_e.
         `roofline_gather` reports the layer-1 gather GEMM the same way.
         `kernels` lists every library call's per-launch time and share of
         the step from the same events.
cpu_baseline: the unmodified reference (scattermlp, vendored to baseline/_ref)
         on the host cores, one fwd+bwd of a bounded sample (T=256 tokens at
         C1 dims), rank 0 at N=1 only (baseline/cpu_reference.py).
--impl reference: the same metric from the unmodified reference on the host
         CPU, --steps steps of T=256 tokens after --warmup untimed ones.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (T, d_model, d_expert, E, k, description)
    "C0": (4096, 512, 1024, 8, 2, "C0 oracle config: T=4096, d_model=512, d_expert=1024, E=8, k=2"),
    "C1": (32768, 4096, 14336, 8, 2,
           "C1 Mixtral-8x7B MLP layer: T=32768, d_model=4096, d_expert=14336, E=8, k=2, gelu, fwd+bwd"),
    "C2": (32768, 4096, 1792, 64, 8,
           "C2 fine-grained: T=32768, d_model=4096, d_expert=1792, E=64, k=8, gelu, fwd+bwd"),
}
METRIC = "SMoE MLP fwd+bwd tokens/sec & TFLOPS (% bf16 peak), Mixtral shape, 1/2/4/8 GPU"


def flops_per_step(T, d, de, E, k):
    return 12.0 * T * k * d * de


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self):
        """Host time at the start/end of the device-timed region (after a synchronize)."""
        return time.perf_counter()

    def stop(self, window=None):
        """Summarise the samples taken inside `window` = (t0, t1) (all samples if None):
        idle samples before the timed region would otherwise pull the median up."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, watts = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for t, ln in self.lines if window is None or window[0] <= t <= window[1] + 0.05]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            try:
                watts.append(float(parts[2]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        watts.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm),
                "power_w": watts[len(watts) // 2] if watts else None}


# ---------------------------------------------------------------------------
# CPU legs: cpu_baseline and --impl reference
#
# Both time the UNMODIFIED reference (scattermlp, installed into baseline/_ref
# by baseline/vendor_reference.py) through its own public API on the host
# cores (baseline/cpu_reference.py: SCATTERMLP_WORKERS = all cores, one BLAS
# thread each — the faster of the reference's two thread configurations at
# C1 dims).  Only if baseline/_ref is absent do they fall back to the oracle
# port (oracle/scattermlp_oracle.py) and say so ("kind": "port").


def cpu_oracle_step_time(T, d, de, E, k, seed=0):
    """One fwd+bwd of the oracle port on T tokens; returns seconds."""
    import numpy as np
    from oracle import scattermlp_oracle as orc

    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (T, d)).astype(np.float32)
    w1 = (rng.uniform(-1, 1, (E, d, de)) / np.sqrt(d)).astype(np.float32)
    w2 = (rng.uniform(-1, 1, (E, de, d)) / np.sqrt(de)).astype(np.float32)
    wg = (rng.uniform(-1, 1, (d, E)) / np.sqrt(d)).astype(np.float32)
    idx, p = orc.topk_routing(orc.gate_probs(x, wg), k)
    dy = rng.uniform(-1, 1, (T, d)).astype(np.float32)

    def step():
        y, st = orc.smoe_mlp_forward(x, w1, w2, idx, p, E)
        orc.smoe_mlp_backward(x, w1, w2, p, st, dy)

    t0 = time.perf_counter()
    step()
    return time.perf_counter() - t0


def cpu_reference(config, tokens, warmup, repeats):
    """dict(value tok/s, ms_per_step, p5/p95, cores, kind, sample) for the CPU reference."""
    from baseline import cpu_reference as cref

    if cref.available():
        r = cref.measure(config, tokens, threads="workers", warmup=warmup, repeats=repeats)
        return {"value": r["tokens_per_s_mean"], "ms_per_step": 1e3 * r["mean_s"],
                "ms_median": 1e3 * r["median_s"], "ms_p5": 1e3 * r["p5_s"], "ms_p95": 1e3 * r["p95_s"],
                "cores": r["cores"], "kind": "reference", "cpu_model": r["cpu_model"],
                "sample": f"T={tokens} tokens at {config} dims per step, {repeats} step(s): the unmodified reference "
                          f"(scattermlp from baseline/_ref, smoe_mlp_forward + smoe_mlp_backward, f32 storage / "
                          f"f64 accumulate), SCATTERMLP_WORKERS={r['cores']}, one BLAS thread per worker"}
    T, d, de, E, k, _ = CONFIGS[config]
    for _ in range(warmup):
        cpu_oracle_step_time(tokens, d, de, E, k)
    times = [cpu_oracle_step_time(tokens, d, de, E, k) for _ in range(max(repeats, 1))]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    times.sort()
    return {"value": tokens * len(times) / sum(times), "ms_per_step": 1e3 * sum(times) / len(times),
            "ms_median": 1e3 * times[len(times) // 2], "ms_p5": 1e3 * times[0], "ms_p95": 1e3 * times[-1],
            "cores": cores, "kind": "port",
            "sample": f"T={tokens} tokens at {config} dims per step (oracle/scattermlp_oracle.py port; "
                      f"baseline/_ref absent)"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path on the host cores."""
    if rank != 0:
        return
    T, d, de, E, k, desc = CONFIGS[args.config]
    r = cpu_reference(args.config, args.ref_tokens, args.warmup, args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "ms_per_step_median": r["ms_median"], "ms_per_step_p5": r["ms_p5"], "ms_per_step_p95": r["ms_p95"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 storage, f64 accumulate",
        "data": "synthetic (the reference's own bench._mlp_problem draws)",
        "config": {"workload": desc, "sample_tokens_per_step": args.ref_tokens},
        "tflops": flops_per_step(args.ref_tokens, d, de, E, k) / (r["ms_per_step"] / 1e3) / 1e12,
        "cpu_baseline": {"value": r["value"], "unit": "tokens/s", "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"], "cpu_model": r.get("cpu_model")},
        "e2e": {"value": r["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg

def _max_over_ranks(v: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2403_08245_b200 as sm
    from paper_2403_08245_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    T, d, de, E, k, desc = CONFIGS[args.config]
    dtype = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = (torch.rand((T, d), generator=g, device=dev) * 2 - 1).to(dtype)
    dy = (torch.rand((T, d), generator=g, device=dev) * 2 - 1).to(dtype)
    if world > 1 and E % world:
        raise SystemExit(f"EP needs num_experts ({E}) divisible by the number of GPUs ({world})")
    e_local = E // world if world > 1 else E
    cfg = sm.SmoeMlpConfig(d_model=d, d_expert=de, num_experts=e_local, k=min(k, e_local))
    w1, w2 = sm.init_smoe_mlp_weights(cfg, 101 + rank, dtype=dtype, device=dev, source="device")
    wg = (torch.rand((d, E), generator=g, device=dev) * 2 - 1) / (d ** 0.5)
    routing = sm.gate_topk(x, wg, k)   # gate GEMM + softmax + top-k in one kernel (router.cu)
    torch.cuda.synchronize()

    ep_mode = args.ep if args.ep != "auto" else ("peer" if world > 1 else "none")
    if ep_mode != "none":
        # expert parallelism: this rank owns experts [rank*E/G, (rank+1)*E/G)
        ep = None
        if ep_mode == "peer":
            # rows stored straight into the owner's buffers over peer memory (ep_peer.py)
            from paper_2403_08245_b200.ep_peer import PeerExpertParallelSmoeMlp
            try:
                ep = PeerExpertParallelSmoeMlp(w1, w2, E, k, max_tokens=T)
            except RuntimeError as exc:   # raised on every rank together
                if rank == 0:
                    print(f"bench: {exc}; falling back to the NCCL exchange", file=sys.stderr)
                ep_mode = "nccl"
        if ep is None:
            from paper_2403_08245_b200.ep import ExpertParallelSmoeMlp
            ep = ExpertParallelSmoeMlp(w1, w2, E)

        def step(xx, dyy, rt, dy_ready=None, on_dx=None):
            y, ctx = ep.forward(xx, rt)
            if dy_ready is not None:
                dy_ready()
            grads = ep.backward(ctx, dyy)
            return y, grads
    else:
        def step(xx, dyy, rt, dy_ready=None, on_dx=None):
            order = sm.compute_grouped_order(rt)
            y, ctx = sm.smoe_mlp_forward(xx, w1, w2, rt, order)
            if dy_ready is not None:   # e2e: dY's H2D copy overlaps the forward
                dy_ready()
            # e2e: dX / dp leave while dW1 computes (the public API's on_dx hook)
            grads = sm.smoe_mlp_backward(ctx, dyy, on_dx=on_dx)
            return y, grads

    def barrier():
        if world > 1:
            dist.barrier()

    # clocks are sampled from the start of the warm-up (the GPU is under the same
    # load there) to the end of the timed steps, so short timed regions still
    # get several nvidia-smi samples; idle time before the warm-up is excluded
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.2)    # nvidia-smi start-up
    torch.cuda.synchronize()
    t_win0 = sampler.mark()
    for _ in range(args.warmup):
        step(x, dy, routing)
    torch.cuda.synchronize()
    barrier()
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one event per step boundary gives the per-step distribution (median / p5 / p95)
    ev_steps = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    from paper_2403_08245_b200.launch_timer import LaunchTimer
    mem_before = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    with LaunchTimer() as lt:   # per-call CUDA events on the launching stream, inside the timed region
        e0.record(st)
        for i in range(args.steps):
            step(x, dy, routing)
            ev_steps[i].record(st)
        e1.record(st)
    torch.cuda.synchronize()
    if ep_mode == "peer":
        ep.check()   # the EP layer's only host read: timeouts / capacity overflow of the timed steps
    # memory of the timed steps alone (before the e2e / roofline sections allocate more)
    peak_step_bytes = torch.cuda.max_memory_allocated(dev)
    step_ms = sorted([e0.elapsed_time(ev_steps[0])] +
                     [ev_steps[i - 1].elapsed_time(ev_steps[i]) for i in range(1, args.steps)])

    def pct(q):
        return step_ms[min(len(step_ms) - 1, int(round(q * (len(step_ms) - 1))))]
    t_win1 = sampler.mark()
    barrier()
    clocks = sampler.stop((t_win0, t_win1))
    clocks["window"] = "warm-up + timed steps"
    per_kernel = lt.summary()
    launches = _lib.launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        ms = _max_over_ranks(ms, dev)
    tokens_total = T * world
    value = tokens_total / (ms / 1e3)
    flops = flops_per_step(T, d, de, E, k)
    peaks, peak_kind = load_peaks()
    tflops_per_gpu = flops / (ms / 1e3) / 1e12

    # ---- e2e through the public API with pinned host buffers --------------
    hx = x.cpu().pin_memory()
    hdy = dy.cpu().pin_memory()
    hidx = routing.expert_idx.cpu().pin_memory()
    hp = routing.p.cpu().pin_memory()
    hdx = torch.empty((T, d), dtype=dtype).pin_memory()
    hdp = torch.empty((T, k), dtype=torch.float32).pin_memory()
    h2d = hx.numel() * hx.element_size() + hdy.numel() * hdy.element_size() + hidx.numel() * 8 + hp.numel() * 4
    d2h = hdx.numel() * hdx.element_size() + hdp.numel() * 4

    # Double-buffered input pipeline, as a training loop would run it: step i+1's
    # H2D copies and step i's D2H copies run on a copy stream while step i
    # computes.  Every step's copies are inside the timed region.
    cs = torch.cuda.Stream(device=dev)        # H2D of the next step's inputs
    cs_out = torch.cuda.Stream(device=dev)    # D2H of this step's results (its own copy engine)
    dbufs = [dict(x=torch.empty_like(x), dy=torch.empty_like(dy), ids=torch.empty_like(routing.expert_idx),
                  p=torch.empty_like(routing.p)) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]      # forward inputs (ids, p, X) landed
    ev_dy = [torch.cuda.Event() for _ in range(2)]      # dY landed (needed only by the backward)
    ev_done = [torch.cuda.Event() for _ in range(2)]

    def prefetch_inputs(slot):
        b = dbufs[slot]
        with torch.cuda.stream(cs):
            cs.wait_event(ev_done[slot])             # the step that last used this slot has finished
            b["ids"].copy_(hidx, non_blocking=True)
            b["p"].copy_(hp, non_blocking=True)
            b["x"].copy_(hx, non_blocking=True)
            ev_in[slot].record(cs)
            b["dy"].copy_(hdy, non_blocking=True)
            ev_dy[slot].record(cs)

    def e2e_run(n_steps):
        for s_ in range(2):
            ev_done[s_].record(st)
        prefetch_inputs(0)
        for i in range(n_steps):
            slot = i % 2
            if i + 1 < n_steps:
                prefetch_inputs(1 - slot)
            st.wait_event(ev_in[slot])
            b = dbufs[slot]
            rt = sm.RoutingResult(expert_idx=b["ids"], p=b["p"], gate_full=routing.gate_full, renormalized=True,
                                  validate=False)
            sent = []

            def send_results(dx_, dp_):
                # D2H of this step's results as soon as they are enqueued
                ev_res = torch.cuda.Event()
                ev_res.record(st)
                with torch.cuda.stream(cs_out):
                    cs_out.wait_event(ev_res)
                    hdx.copy_(dx_, non_blocking=True)
                    hdp.copy_(dp_, non_blocking=True)
                    dx_.record_stream(cs_out)
                    dp_.record_stream(cs_out)
                sent.append(True)

            _, grads = step(b["x"], b["dy"], rt, dy_ready=lambda: st.wait_event(ev_dy[slot]), on_dx=send_results)
            ev_done[slot].record(st)
            if not sent:   # paths without the hook (expert-parallel): after the step
                send_results(grads.dx, grads.dp)
        st.wait_stream(cs)
        st.wait_stream(cs_out)

    e2e_run(max(2, args.warmup))
    torch.cuda.synchronize()
    barrier()
    e0.record(st)
    e2e_run(args.steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1) / args.steps
    if world > 1:
        ms_e2e = _max_over_ranks(ms_e2e, dev)

    kernels = {lab: {"launches_per_step": d["launches"] / args.steps, "ms_per_launch": d["ms_per_launch"],
                     "share_of_step": d["ms_total"] / args.steps / ms}
               for lab, d in per_kernel.items()}
    # the layer-1 GEMM's label (the routing-weight-scaled MLP path appends " scaled")
    L1_LABEL = next((lab for lab in kernels if lab.startswith("scatter2scatter S->G +act(pre,post)")),
                    "scatter2scatter S->G +act(pre,post)")

    # ---- roofline: dominant kernel (layer-1 forward grouped GEMM) ----
    # achieved = its algorithmic FLOPs / its mean launch duration inside the
    # timed steps (events on its stream); it is also timed alone for reference.
    if ep_mode != "none":
        # this rank's local experts only (the EP shard)
        kk = min(k, e_local)
        rt_local = sm.topk_select(torch.softmax(torch.randn(T, e_local, device=dev, generator=g), 1), kk)
        order = sm.compute_grouped_order(rt_local)
    else:
        kk = k
        order = sm.compute_grouped_order(routing)
    n = T * kk
    h_pre = torch.empty((n, de), dtype=dtype, device=dev)
    h = torch.empty_like(h_pre)
    reps = 10

    def l1():
        sm.scatter2scatter(x, w1, order, kk, sm.SCATTERED_TO_GROUPED, out=h_pre, activation="gelu", act_out=h)

    for _ in range(2):
        l1()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        l1()
    e1.record(st)
    torch.cuda.synchronize()
    ms_l1_alone = e0.elapsed_time(e1) / reps
    l1_flops = 2.0 * n * d * de
    ms_l1 = kernels[L1_LABEL]["ms_per_launch"] if (world == 1 and L1_LABEL in kernels) else ms_l1_alone
    traffic_db = {}
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            traffic_db = json.loads(tfile.read_text())
        except Exception:
            traffic_db = {}

    def roof(label, ms_launch, desc, timed):
        achieved = l1_flops / (ms_launch / 1e3) / 1e12     # every GEMM of the step is 2*n*d*d_e FLOP
        # Kernels timed inside the long step are compared with the sustained peak (the
        # profiling recipe's rule); a kernel timed alone with the burst peak.
        sustained = timed == in_step and "bf16_tflops_sustained" in peaks
        pk = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
        return {"bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                "frac": achieved / pk, "frac_of_burst": achieved / peaks["bf16_tflops"],
                "traffic": traffic_db.get(f"{args.config}:{label}"),
                "kernel": desc, "label": label,
                "algorithmic": f"2*T*k*d_model*d_expert = {l1_flops:.4g} FLOP per launch",
                "ms_per_launch": ms_launch, "share_of_step": kernels.get(label, {}).get("share_of_step"),
                "timed": timed, "peak_kind": f"{peak_kind} {'sustained' if sustained else 'burst'}"}

    in_step = "inside the timed steps (CUDA events around each launch on its stream)"
    gather_roof = roof(L1_LABEL, ms_l1, "scatter2scatter S->G layer-1 fwd (cp.async row gather + grouped GEMM + "
                       "fused GELU epilogue)", in_step if world == 1 else "alone (10 back-to-back launches)")
    gather_roof["ms_per_launch_alone"] = ms_l1_alone
    gemms = {lab: v for lab, v in kernels.items() if lab.startswith(("scatter2scatter", "group_xty"))}
    if world == 1 and gemms:
        # the dominant kernel = the GEMM family with the largest share of the step
        dom = max(gemms, key=lambda lab: gemms[lab]["share_of_step"])
        dom_desc = ("group_xty: grouped-K tcgen05 GEMM (dW = Xg^T Yg per expert bin; 2 launches per step)"
                    if dom.startswith("group_xty") else f"{dom} (tcgen05 grouped GEMM)")
        roofline = roof(dom, gemms[dom]["ms_per_launch"], dom_desc, in_step)
    else:
        roofline = gather_roof

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(args.config, args.ref_tokens, 0, 1)
        cpu_baseline = {"value": r["value"], "unit": "tokens/s", "cores": r["cores"], "kind": r["kind"],
                        "sample": r["sample"] + f"; {r['ms_per_step'] / 1e3:.1f} s", "cpu_model": r.get("cpu_model")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, softmax top-k routing)",
            "config": {"workload": desc, "global_batch": T * world, "seq_len": None,
                       "parallelism": (f"ep{world} (experts sharded; " + ("rows stored into the owners' buffers over "
                                       "peer memory, ep_peer.py)" if ep_mode == "peer" else
                                       "NCCL all-to-all-v dispatch/combine, ep.py)")) if ep_mode != "none"
                       else "single GPU",
                       "l2": "inputs larger than L2 (W1+W2 1.9 GB, H 1.9 GB); no flush",
                       "engine": sm.get_engine(), "timed": "flatten_and_sort + smoe_mlp_forward + smoe_mlp_backward"},
            "tflops_per_gpu": tflops_per_gpu,
            "pct_bf16_peak": tflops_per_gpu / peaks["bf16_tflops"],
            "pct_bf16_peak_sustained": tflops_per_gpu / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
            "e2e": {"value": tokens_total / (ms_e2e / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
            "gpu_launches": launches,
            "roofline": roofline,
            "roofline_gather": gather_roof,
            # expert parallel: share of the step in exchange-only calls (dispatch
            # stores, count exchange, completion barriers, dp return); the returns
            # ride in the GEMM epilogues (ep_gemm_return) and are not counted here
            "ep_exchange_share_of_step": (sum(v["share_of_step"] for lab, v in kernels.items()
                                              if lab.startswith(("ep_dispatch", "ep_sync", "ep_put", "ep_dp_return",
                                                                 "ep_return")))
                                          if ep_mode == "peer" else None),
            "kernels": kernels,
            "cpu_baseline": cpu_baseline,
            "clocks": clocks,
            "step_ms": {"median": pct(0.5), "p5": pct(0.05), "p95": pct(0.95), "mean": ms,
                        "n": len(step_ms), "timing": "CUDA events at every step boundary on the launching stream"},
            # peak over the timed steps only: inputs + weights + the step's working set;
            # the e2e buffers and the roofline section allocate after this is read
            "peak_memory_gb": peak_step_bytes / 1e9,
            "memory": {"resident_before_steps_gb": mem_before / 1e9, "peak_during_steps_gb": peak_step_bytes / 1e9,
                       "step_working_set_gb": (peak_step_bytes - mem_before) / 1e9},
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 100 on the GPU; 3 for --impl reference, ~10 s each)")
    ap.add_argument("--warmup", type=int, default=None,
                    help="untimed warm-up steps (default 10 on the GPU; 1 for --impl reference)")
    ap.add_argument("--config", default="C1", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-tokens", type=int, default=256,
                    help="tokens per CPU reference step (a bounded sample of the workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", default=None)
    ap.add_argument("--ep", default="auto", choices=["auto", "peer", "nccl", "none"],
                    help="expert-parallel exchange (auto: peer memory when N>1, none at N=1; "
                         "peer/nccl at N=1 time the EP path on one GPU)")
    args = ap.parse_args()
    cpu_arm = args.impl == "reference"
    if args.steps is None:
        args.steps = 3 if cpu_arm else 100
    if args.warmup is None:
        args.warmup = 1 if cpu_arm else 10
    args.warmup = max(args.warmup, 0)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # Test rig only (SMOE_BENCH_SHARE_GPU=1): every rank on GPU 0 with gloo for
    # the host collectives, so the N>1 code path (peer-memory EP over CUDA IPC,
    # max-over-ranks timing) runs on a one-GPU box.  Its timings are meaningless.
    share_gpu = os.environ.get("SMOE_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local_rank = 0

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    if args.engine:
        import paper_2403_08245_b200 as sm
        sm.set_engine(args.engine)
    if world > 1 or args.ep in ("peer", "nccl"):
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
