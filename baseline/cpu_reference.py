"""Time the unmodified reference (scattermlp, vendored in baseline/_ref) on the host CPU.

SURVEY.md §8(d) CPU protocol, on the reference's own public API and stock code
path: ``smoe_mlp_forward(training=True)`` + ``smoe_mlp_backward`` on the
problem its bench builds (``bench._mlp_problem``, bench.py:120-130), timed
with its own ``time_callable`` (median / p5 / p95, bench.py:86-100).  Nothing
from this repository runs on that path.

The thread configuration must be fixed before NumPy loads, so every
measurement runs in a fresh interpreter:

  blas    : OPENBLAS_NUM_THREADS = all cores, SCATTERMLP_WORKERS = 1
  workers : OPENBLAS_NUM_THREADS = 1,         SCATTERMLP_WORKERS = all cores

    python baseline/cpu_reference.py --config C1 --tokens 256 --threads blas
    python baseline/cpu_reference.py --sweep          # the full §8(d) table

Prints one JSON object per measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"

DIMS = {  # name: (d_model, d_expert, E, k, full T)
    "C0": (512, 1024, 8, 2, 4096),
    "C1": (4096, 14336, 8, 2, 32768),
    "C2": (4096, 1792, 64, 8, 32768),
}


def available() -> bool:
    return (REF / "scattermlp" / "__init__.py").exists()


def cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def thread_env(mode: str) -> dict:
    n = str(cores())
    env = dict(os.environ)
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[var] = n if mode == "blas" else "1"
    env["SCATTERMLP_WORKERS"] = "1" if mode == "blas" else n
    return env


def _measure_in_process(config: str, tokens: int, warmup: int, repeats: int, seed: int) -> dict:
    sys.path.insert(0, str(REF))
    import scattermlp
    from scattermlp import bench

    assert Path(scattermlp.__file__).resolve().is_relative_to(REF.resolve()), scattermlp.__file__
    d, de, e, k, _ = DIMS[config]
    t_build = time.perf_counter()
    _, x, w1, w2, routing, order = bench._mlp_problem(d, de, e, k, tokens, seed)
    dy = scattermlp.seeded_random_matrix(tokens, d, seed + 13, scale=1.0)
    t_build = time.perf_counter() - t_build

    def step():
        y, ctx = scattermlp.smoe_mlp_forward(x, w1, w2, routing, order, training=True)
        scattermlp.smoe_mlp_backward(ctx, dy)

    # the reference's own protocol (bench.time_callable, bench.py:86-100) plus the mean
    samples = []

    def timed():
        t0 = time.perf_counter_ns()
        step()
        samples.append(time.perf_counter_ns() - t0)

    med, p5, p95 = bench.time_callable(timed, warmup, repeats)
    samples = samples[max(warmup, 0):]
    mean_s = sum(samples) / len(samples) * 1e-9
    return {"config": config, "tokens": tokens, "median_s": med * 1e-9, "p5_s": p5 * 1e-9, "p95_s": p95 * 1e-9,
            "mean_s": mean_s, "tokens_per_s": tokens / (med * 1e-9), "tokens_per_s_mean": tokens / mean_s,
            "repeats": repeats, "warmup": warmup,
            "problem_build_s": t_build, "flops_per_step": 12.0 * tokens * k * d * de,
            "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
            "scattermlp_workers": os.environ.get("SCATTERMLP_WORKERS")}


def measure(config: str, tokens: int, threads: str = "blas", warmup: int = 1, repeats: int = 3,
            seed: int = 0, timeout: float = 1800.0) -> dict:
    """One measurement in a fresh interpreter with the thread configuration applied."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--config", config, "--tokens", str(tokens),
           "--threads", threads, "--warmup", str(warmup), "--repeats", str(repeats), "--seed", str(seed),
           "--in-process"]
    res = subprocess.run(cmd, env=thread_env(threads), capture_output=True, text=True, timeout=timeout)
    if res.returncode != 0:
        raise RuntimeError(f"reference CPU run failed:\n{res.stderr[-3000:]}")
    out = json.loads(res.stdout.strip().splitlines()[-1])
    out.update(threads=threads, cores=cores(), cpu_model=cpu_model(), kind="reference",
               impl="scattermlp 0.1.0 from baseline/_ref (unmodified)")
    return out


def sweep(repeats: int = 3) -> list[dict]:
    """§8(d): C0 at full size, C1 / C2 dims at T in {256, 1024}; both thread configurations."""
    rows = []
    for config, tokens in (("C0", 4096), ("C1", 256), ("C1", 1024), ("C2", 256), ("C2", 1024)):
        for threads in ("blas", "workers"):
            row = measure(config, tokens, threads, warmup=1, repeats=repeats)
            print(json.dumps(row), flush=True)
            rows.append(row)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1", choices=sorted(DIMS))
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--threads", default="blas", choices=["blas", "workers"])
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--in-process", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if not available():
        raise SystemExit("baseline/_ref/scattermlp missing: run python baseline/vendor_reference.py")
    if args.in_process:
        print(json.dumps(_measure_in_process(args.config, args.tokens, args.warmup, args.repeats, args.seed)))
    elif args.sweep:
        sweep(args.repeats)
    else:
        print(json.dumps(measure(args.config, args.tokens, args.threads, args.warmup, args.repeats, args.seed)))


if __name__ == "__main__":
    main()
