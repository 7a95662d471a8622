"""Energy per launch of each C1 GEMM mode under the power cap.

Runs one mode back to back for a few seconds (steady state, power-capped),
samples nvidia-smi power / SM clock meanwhile, and reports ms per launch,
median SM MHz, median W, and J per launch / TFLOP per J.  The bench step is
power-capped (sw_power_cap), so energy per FLOP — not tensor-pipe activity at
a fixed clock — is what sets its speed.

usage: python scripts/energy.py [mode ...]   (modes as in prof_one.py)
"""
import json
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402

T, d, de, E, k = 32768, 4096, 14336, 8, 2
n = T * k
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
x = (torch.rand(T, d, device=dev, generator=g) * 2 - 1).bfloat16()
xg = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).bfloat16()
w = ((torch.rand(E, d, de, device=dev, generator=g) * 2 - 1) / d ** 0.5).bfloat16()
routing = sm.topk_select(torch.softmax(torch.randn(T, E, device=dev, generator=g), 1), k)
order = sm.compute_grouped_order(routing)
h = ((torch.rand(n, de, device=dev, generator=g) * 2 - 1) * 0.5).bfloat16()
h2 = torch.empty_like(h)

MODES = {
    "l1": lambda: sm.scatter2scatter(x, w, order, k, sm.SCATTERED_TO_GROUPED, out=h2, activation="gelu", act_out=h2),
    "gather": lambda: sm.scatter2scatter(x, w, order, k, sm.SCATTERED_TO_GROUPED, out=h2),
    "rows": lambda: sm.scatter2scatter(xg, w, order, 1, sm.GROUPED_TO_GROUPED, out=h2),
    "l2": lambda: sm.scatter2scatter(h, w.view(E, de, d), order, 1, sm.GROUPED_TO_SCATTERED, out=xg),
    "dh": lambda: sm.scatter2scatter(xg, w.view(E, de, d), order, 1, sm.GROUPED_TO_GROUPED, transpose_w=True, out=h2,
                                     activation="gelu", act_grad_of=h),
    "dx": lambda: sm.scatter2scatter(h, w, order, 1, sm.GROUPED_TO_SCATTERED, transpose_w=True, out=xg),
    "xty": lambda: sm.group_xty(h, xg, order),
    "cublas": lambda: torch.matmul(xg, w[0]),   # dense reference: n x d @ d x d_e (same FLOPs as one GEMM)
    "cublas_dw": lambda: torch.matmul(xg.t(), h),   # dense dW-shaped reference: d x n @ n x d_e (K = n)
    "cublas_l2": lambda: torch.matmul(h, w.view(E, de, d)[0]),   # n x d_e @ d_e x d (K = d_e)
    # torch's grouped GEMM (vendor kernels) on the exact grouped problems: layer 2 (K = d_e)
    # and the grouped-input K = d GEMM, expert bins from the same routing
    "gmm_l2": lambda: torch._grouped_mm(h, w.view(E, de, d), offs=order.bin_offsets[1:]),
    "gmm_rows": lambda: torch._grouped_mm(xg, w, offs=order.bin_offsets[1:]),
}


def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    for line in p.stdout:
        if stop.is_set():
            break
        try:
            a, b = (float(v) for v in line.split(","))
            out.append((a, b))
        except ValueError:
            pass
    p.terminate()


def main():
    modes = sys.argv[1:] or list(MODES)
    flop = 2.0 * n * d * de
    for m in modes:
        fn = MODES[m]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        samples, stop = [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, samples), daemon=True)
        th.start()
        time.sleep(0.5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 0
        t0 = time.time()
        e0.record()
        while time.time() - t0 < 4.0:
            for _ in range(10):
                fn()
            reps += 10
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        ms = e0.elapsed_time(e1) / reps
        steady = samples[len(samples) // 3:] or samples
        watts = sorted(s[0] for s in steady)
        mhz = sorted(s[1] for s in steady)
        w_med = watts[len(watts) // 2] if watts else float("nan")
        j = w_med * ms / 1e3
        print(json.dumps({"mode": m, "ms_per_launch": ms, "sm_mhz": mhz[len(mhz) // 2] if mhz else None,
                          "power_w": w_med, "joule_per_launch": j, "tflop_per_joule": flop / j / 1e12,
                          "tflops": flop / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
