"""Benchmark: rank-k accelerated RPCholesky wall time on B200 (BASELINE.json metric).

A step is one full factorization (accelerated_rpcholesky over the C-ABI) of the
configured workload.  Default workload: config C4 of BASELINE.json (N=1e6,
d=30 anisotropic Gaussian data, Gaussian kernel sigma=3, k=1000, b=120, seed 0),
the configuration the metric names.  Points are synthetic and seeded
(paper_2410_03969_b200/workloads.py); no dataset is involved.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

value       : device wall time (s) of one factorization with the points resident in HBM
              (CUDA events, max over ranks); lower is better
e2e         : same call through the host C-ABI entry (host X in, pinned) plus the
              device->host copy of the full factor, pivots and chol_factor
roofline    : the fused K5+K6 update kernel (FP64 DMMA bound) against the FP64
              tensor peak measured on this pool (profiles/r01_fp64_peaks.json)
cpu_baseline: the CPU oracle restatement timed on this host on a bounded sample
--impl reference: the reference path's CPU implementation (oracle port, all host
              threads) on the same config, extrapolated from a bounded sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rank-k RPCholesky wall time (s) & kernel-col GB/s, N=1e6 k=1000, 1/2/4/8 B200"


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 10 ms) during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                    "sw_power_cap": 0x4}
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, [k for k, b in bits.items() if r & b]))
                self._stop.wait(0.01)
        except Exception as e:  # NVML unavailable: fall back to one nvidia-smi reading
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                sm, mx = [float(v) for v in out.split(",")]
                self.samples.append((sm, mx, ["nvml_unavailable:" + type(e).__name__]))
            except Exception:
                pass

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({r for s in self.samples for r in s[2]}),
                "samples": len(self.samples)}


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
    try:
        d = json.load(open(p))
        return float(d["fp64_dmma_tflops"]), "profiles/r01_fp64_peaks.json (tools/fp64_peaks.cu, DMMA, this pool)"
    except Exception:
        return 37.1, "fallback 37.1 TF/s (DMMA measured on this pool, round 1)"


def ncu_traffic(config_name):
    p = os.path.join(ROOT, "profiles", f"update_traffic_{config_name}.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def cpu_sample(w, threads: int, n_sample: int, lowmem: bool = False):
    """Oracle restatement (oracle/, test infrastructure) on N' = n_sample points of
    the same workload; returns (seconds at N', extrapolated seconds at N)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    x = w.points(n_sample)
    o = po.Oracle(x=x, kernel=w.kernel, sigma=w.sigma, n_threads=threads)
    fn = po.accelerated_rpcholesky_lowmem if lowmem else po.accelerated_rpcholesky
    t0 = time.perf_counter()
    fn(o, block_size=w.b, target_rank=w.k, seed=w.seed)
    dt = time.perf_counter() - t0
    return dt, dt * (w.n / n_sample)


def reference_arm(w, args):
    """The reference's own CPU accelerated_rpcholesky: its headers compiled against the
    Eigen-API shim (oracle/_ref, built where /root/reference exists; prebuilt .so here),
    single-threaded as the reference's KernelOracle path is (one 256-wide panel).  Each
    step runs a bounded sample: the first N' rows of the workload with the same k, b, seed;
    the value is scaled by N/N' (the path is linear in N at fixed k).  Falls back to the C
    restatement when the reference build is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    n_sample = args.cpu_sample or min(w.n, 20_000)
    x = w.points(n_sample)
    try:
        import pyref
        use_ref = pyref.available()
    except Exception:
        use_ref = False
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if use_ref:
            pyref.accelerated_rpcholesky_kernel(x, w.kernel, w.sigma, block_size=w.b,
                                                target_rank=w.k, seed=w.seed)
        else:
            import pyoracle as po
            po.accelerated_rpcholesky(po.Oracle(x=x, kernel=w.kernel, sigma=w.sigma, n_threads=1),
                                      block_size=w.b, target_rank=w.k, seed=w.seed)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    dt = statistics.median(times)
    v = dt * (w.n / n_sample)
    kind = "reference" if use_ref else "port"
    cpu = {"value": v, "unit": "s", "cores": 1, "kind": kind,
           "sample": (f"{'reference headers (oracle/_ref, Eigen-API shim)' if use_ref else 'C restatement'}"
                      f" single-threaded on the first N'={n_sample} rows of {w.name} (same k/b/seed): "
                      f"{dt:.2f} s median of {len(times)}, x N/N'={w.n / n_sample:g}")}
    return v, cpu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="N' for the CPU sample (0=auto)")
    ap.add_argument("--variant", default="standard", choices=["standard", "lowmem"],
                    help="lowmem: accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485)")
    args = ap.parse_args()

    from paper_2410_03969_b200 import workloads
    w = workloads.CONFIGS[args.config]
    rank, world, local_rank = env_rank()
    n_cores = os.cpu_count() or 1
    cfg_json = {"workload": f"{w.name}: {w.kernel} N={w.n} d={w.d} sigma={w.sigma:.6g} "
                            f"k={w.k} b={w.b} seed={w.seed}",
                "n": w.n, "d": w.d, "k": w.k, "b": w.b, "kernel": w.kernel,
                "parallelism": f"row-shard{world}" if world > 1 else "single-gpu",
                "l2": "inputs larger than L2 (F alone is >= 1.8 GB at C2-C5)"}
    lowmem = args.variant == "lowmem"
    if lowmem:
        cfg_json["variant"] = "lowmem (no N x k factor; A(R, S_all) regenerated per round)"
        cfg_json["l2"] = "X and u larger than L2 at C2-C5; the kernel block never leaves the SM"

    if args.impl == "reference":
        if rank != 0:
            return
        v, cpu = reference_arm(w, args)
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": cfg_json, "cpu_baseline": cpu,
                          "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    import torch
    from paper_2410_03969_b200 import api
    from paper_2410_03969_b200 import _lib as L
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(api.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        ctx = api.Context(local_rank, nccl_id=bytes(idt.cpu().numpy().tobytes()), nranks=world,
                          rank=rank)
    else:
        dist = None
        ctx = api.Context(local_rank)

    x = w.points()                                   # host, row-major N x d
    r0, nr = ctx.shard_rows(w.n)
    x_dev = torch.from_numpy(np.ascontiguousarray(x[r0:r0 + nr])).to(dev)
    spec = api.KernelSpec(w.kernel, w.sigma)
    cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def one_step():
        fn = api.accelerated_rpcholesky_lowmem_device if lowmem else api.accelerated_rpcholesky_device
        return fn(x_dev.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR, spec, cfg, ctx)

    for _ in range(args.warmup):
        one_step().free()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record()
        for _ in range(args.steps):
            r = one_step()
            results.append((r.timing, r.rank, [len(a) for a in r.accepted], r.relative_trace_error))
            r.free()
        ev1.record()
        barrier()
    total_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    sec_per_step = total_ms / args.steps / 1e3
    timing, k_final, m_seq, trace_err = results[-1]
    upd_ms = timing["update_ms"]
    flops = timing["update_flops"]
    peak, peak_src = fp64_peak()
    achieved = flops / (upd_ms * 1e-3) / 1e12 if upd_ms > 0 else 0.0
    tr = ncu_traffic(w.name + ("_lowmem" if lowmem else ""))
    traffic = tr["bytes_per_launch_mean"] if tr else None
    traffic_note = tr.get("note") if tr else None

    # kernel-col GB/s: standalone K5 on this run's accepted blocks (rank 0 only)
    col_gbs = None
    if rank == 0 and world == 1 and not lowmem:
        rr = one_step()
        ko = api.KernelOracle(x, spec)
        tot_ms, cols_total = 0.0, 0
        for acc in rr.accepted:
            if len(acc) == 0:
                continue
            ko.columns(acc, ctx)  # warm-up: first launch of a kernel variant loads its module
            _, ms = ko.columns(acc, ctx, return_ms=True)
            tot_ms += ms
            cols_total += len(acc)
        rr.free()
        col_gbs = 8.0 * w.n * cols_total / (tot_ms * 1e-3) / 1e9 if tot_ms > 0 else None

    # e2e through the host C-ABI: host X (pinned) in, full factor + pivots + chol out
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
        cap = api.factor_capacity(w.n, cfg)
        fout = torch.empty((nr * cap + cap * cap + nr + 16,),
                           dtype=torch.float64).pin_memory().numpy()
        ko = api.KernelOracle(xh, spec)
        e2e_times = []
        for i in range(1 + min(args.steps, 3)):
            barrier()
            t0 = time.perf_counter()
            import ctypes as C
            lib = L.load()
            if lowmem:  # LowMemResult: chol_factor + residual diagonal out
                res = api.accelerated_rpcholesky_lowmem(ko, cfg, ctx)
                kk = res.rank
                L.check(lib.rpc_result_chol_copy(res._handle, C.c_void_p(fout.ctypes.data)),
                        ctx.handle)
                L.check(lib.rpc_result_residual_diag_copy(
                    res._handle, C.c_void_p(fout.ctypes.data + 8 * (kk * kk - r0))), ctx.handle)
            else:
                # the factor streams into this rank's pinned rows (ld = nr, global row
                # indexing) while the rounds run; then chol_factor; pivots come with the handle
                xx, lay, ldx = ko._host_layout()
                h = C.c_void_p()
                L.check(lib.rpc_accelerated_rpcholesky_into(
                    ctx.handle, xx.ctypes.data, w.n, w.d, ldx, lay, ko._c_spec(), cfg.to_c(),
                    C.c_void_p(fout.ctypes.data - r0 * 8), nr, cap, C.byref(h)), ctx.handle)
                res = api._wrap_result(h, ctx)
                kk = res.rank
                L.check(lib.rpc_result_chol_copy(res._handle,
                                                 C.c_void_p(fout.ctypes.data + 8 * nr * cap)),
                        ctx.handle)
            barrier()
            dt = time.perf_counter() - t0
            res.free()
            if i > 0:
                e2e_times.append(dt)
        tt = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        d2h = (k_final * k_final * 8 + nr * 8 + k_final * 8) if lowmem else \
            (nr * k_final * 8 + k_final * 8 + k_final * k_final * 8)
        e2e = {"value": float(tt.item()), "unit": "s",
               "h2d_bytes_per_step": int(nr * w.d * 8), "d2h_bytes_per_step": int(d2h)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_sample = args.cpu_sample or min(w.n, 10_000 if lowmem else 100_000)
        dt, ext = cpu_sample(w, n_cores, n_sample, lowmem)
        cpu = {"value": ext, "unit": "s", "cores": n_cores, "kind": "port",
               "sample": f"oracle restatement on the first N'={n_sample} rows of {w.name}, same "
                         f"k/b/seed, {dt:.2f} s measured, x N/N' to the full N"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": sec_per_step, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec_per_step * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads.py)", "config": cfg_json,
            "kernel_col_gbs": col_gbs,
            "rank_final": k_final, "rounds": len(m_seq), "accepted_per_round": m_seq,
            "relative_trace_error": trace_err,
            "device_factorize_ms": timing["factorize_ms"],
            "host_ms": {k: round(timing[k], 3) for k in ("host_total_ms", "host_setup_ms",
                                                         "host_loop_ms", "host_final_ms",
                                                         "upload_ms")},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "kernel": ("lowmem_kernel (A(R, S_all) regenerated in SMEM + FP64 DMMA GEMM with "
                                    "the new L^-1 rows + diag update)") if lowmem else
                                   "update_kernel (fused K5 kernel columns + K6 FP64 DMMA GEMM + L^-T + diag update)",
                         "traffic_note": traffic_note,
                         "peak_source": peak_src,
                         "per_launch_flops": flops / max(1, timing["update_launches"]),
                         "update_ms_per_step": upd_ms,
                         "update_share_of_step": upd_ms / (sec_per_step * 1e3)},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(timing["kernel_launches"]) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
