"""Benchmark: rank-k accelerated RPCholesky wall time on B200 (BASELINE.json metric).

A step is one full factorization (accelerated_rpcholesky over the C-ABI) of the
configured workload.  Default workload: config C4 of BASELINE.json (N=1e6,
d=30 anisotropic Gaussian data, Gaussian kernel sigma=3, k=1000, b=120, seed 0),
the configuration the metric names.  Points are synthetic and seeded
(paper_2410_03969_b200/workloads.py); no dataset is involved.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

--gpus N    : without torchrun, spawns N ranks (one process per GPU, NCCL, row-sharded);
              under torchrun (WORLD_SIZE set) each process is one rank
value       : device wall time (s) of one factorization with the points resident in HBM
              (CUDA events per step, median over the K steps, max over ranks)
e2e         : same call through the host C-ABI entry (host X in, pinned) plus the
              device->host copy of the full factor, pivots and chol_factor
roofline    : the fused K5+K6 update kernel (FP64 DMMA bound) against the FP64
              tensor peak measured on this pool (profiles/r01_fp64_peaks.json)
parity      : after the timed region, the full workload is factored by the CPU restatement
              of the reference (oracle/, all host threads) and compared with the GPU result
              in fast (benched) and replay mode: pivots, trace, ||dF||/||F||, trace error,
              the oracle's decision margins
cpu_baseline: that same oracle run on the full workload (no extrapolation)
--impl reference: the reference's own CPU code (oracle/_ref: its headers compiled against
              the Eigen-API shim, single thread as its path runs) on a bounded sample of the
              workload (first N'=1e5 rows, same k/b/seed), scaled by N/N'; the line declares
              the extrapolation and quotes the committed full-N calibration
              (profiles/r02_reference_calibration_<config>.json, tools/reference_calibration.py)
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


def int8_peak():
    """Dense int8 tensor peak: twice the measured dense bf16 GEMM rate (B200 runs int8/fp8 at 2x
    bf16 dense), from the driver-written MEASURED_PEAKS.json; else the nominal 4500 TOP/s."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return 2.0 * float(d["bf16_tflops"]), "2 x MEASURED_PEAKS.json bf16_tflops (burst, dense)"
    except Exception:
        return 4500.0, "nominal B200 dense int8 (4.5 POP/s)"


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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_arm(w, args):
    """The reference's own CPU accelerated_rpcholesky: its headers compiled against the
    Eigen-API shim (oracle/_ref, built where /root/reference exists; prebuilt .so here),
    single-threaded as the reference's KernelOracle path is (one 256-wide panel, Eigen
    without OpenMP).  Each step runs a bounded sample: the first N' rows of the workload
    with the same k, b, seed; the value is scaled by N/N' (the path is linear in N at fixed
    k: residual GEMM, TRSM and kernel columns are all O(N)).  A CPU path has no warm-up
    state, so at most one warm-up sample runs.  Falls back to the C restatement when the
    reference build is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    n_sample = args.cpu_sample or min(w.n, 100_000)
    x = w.points(n_sample)
    try:
        import pyref
        use_ref = pyref.available()
    except Exception:
        use_ref = False
    times = []
    warm = min(args.warmup, 1)
    for i in range(warm + args.steps):
        t0 = time.perf_counter()
        if use_ref:
            pyref.accelerated_rpcholesky_kernel(x, w.kernel, w.sigma, block_size=w.b,
                                                target_rank=w.k, seed=w.seed)
        else:
            import pyoracle as po
            po.accelerated_rpcholesky(po.Oracle(x=x, kernel=w.kernel, sigma=w.sigma, n_threads=1),
                                      block_size=w.b, target_rank=w.k, seed=w.seed)
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
    dt = statistics.median(times)
    factor = w.n / n_sample
    v = dt * factor
    kind = "reference" if use_ref else "port"
    calib = None
    cp = os.path.join(ROOT, "profiles", f"r02_reference_calibration_{w.name}.json")
    if os.path.exists(cp):
        c = json.load(open(cp))
        calib = {"measured_full_n_s": c.get("full_n_s"), "cpu_model": c.get("cpu_model"),
                 "sample_extrapolated_s": c.get("extrapolated_s"),
                 "extrapolation_over_measured": c.get("extrapolation_over_measured"),
                 "file": os.path.relpath(cp, ROOT)}
    cpu = {"value": v, "unit": "s", "cores": 1, "kind": kind,
           "cpu_model": cpu_model(), "nproc": os.cpu_count(),
           "sample": (f"{'reference headers (oracle/_ref, Eigen-API shim)' if use_ref else 'C restatement'}"
                      f" single-threaded on the first N'={n_sample} rows of {w.name} (same k/b/seed): "
                      f"{dt:.2f} s median of {len(times)} (warm-up {warm}), x N/N'={factor:g}"),
           "extrapolation": {"n_sample": n_sample, "factor": factor, "sample_median_s": dt,
                             "calibration": calib}}
    return v, cpu


def same_run_parity(w, x, spec, cfg_base, ctx, x_dev, threads):
    """SURVEY §8(d) "Parity checks (same run)": the full workload through the CPU restatement
    of the reference (oracle/, test infrastructure, the checker) against the GPU result in
    fast (benched) and replay mode.  Returns (parity dict, oracle seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_2410_03969_b200 import api
    from paper_2410_03969_b200 import _lib as L
    o = po.Oracle(x=x, kernel=w.kernel, sigma=w.sigma, n_threads=threads)
    po.margins_reset(True)
    t0 = time.perf_counter()
    r = po.accelerated_rpcholesky(o, block_size=w.b, target_rank=w.k, seed=w.seed,
                                  copy_factor=False)
    t_cpu = time.perf_counter() - t0
    mg = po.margins_get()
    po.margins_reset(False)
    err_o = po.relative_trace_error(o, r.factor)
    out = {"oracle": f"C restatement (oracle/rpc_oracle.c), {threads} threads, full workload",
           "oracle_s": round(t_cpu, 3), "min_draw_margin": mg.min_draw,
           "min_sweep_margin": mg.min_sweep, "draws": mg.n_draws, "decisions": mg.n_decisions}
    for mode in ("fast", "replay"):
        cfg = api.RunConfig(**{**cfg_base.__dict__, "replay_scan": mode == "replay"})
        g = api.accelerated_rpcholesky_device(x_dev.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR,
                                              spec, cfg, ctx)
        try:
            piv = bool(np.array_equal(g.pivots, r.pivots))
            tr = (len(g.proposed) == len(r.proposed)
                  and all(np.array_equal(a, b) for a, b in zip(g.proposed, r.proposed))
                  and all(np.array_equal(a, b) for a, b in zip(g.accepted, r.accepted)))
            rec = {"pivots_equal": piv, "trace_equal": bool(tr),
                   "trace_diff": abs(g.relative_trace_error - err_o),
                   "factorize_ms": g.timing["factorize_ms"]}
            if piv:
                f = g.factor_into(np.empty((w.n, g.rank), order="F"))
                num = den = 0.0
                for j in range(0, g.rank, 64):
                    dd = f[:, j:j + 64] - r.factor[:, j:j + 64]
                    num += float(np.einsum("ij,ij->", dd, dd))
                    rr = r.factor[:, j:j + 64]
                    den += float(np.einsum("ij,ij->", rr, rr))
                del f
                rec["f_rel"] = (num / den) ** 0.5
            rec["ok"] = bool(piv and tr and rec.get("f_rel", 1.0) <= 1e-10
                             and rec["trace_diff"] <= 1e-8)
            out[mode] = rec
        finally:
            g.free()
    return out, t_cpu


def spawn_ranks(args) -> int:
    """--gpus N without torchrun: one process per GPU (RANK / LOCAL_RANK / WORLD_SIZE /
    MASTER_* as torchrun sets them); rank 0 prints the JSON line."""
    import socket
    import torch
    n = args.gpus
    if torch.cuda.device_count() < n:
        print(f"bench.py --gpus {n}: only {torch.cuda.device_count()} CUDA device(s) visible",
              file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


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
    ap.add_argument("--no-parity", action="store_true", help="skip the same-run oracle parity")
    args = ap.parse_args()
    if args.impl == "b200" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

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
                          "n_gpus": max(world, args.gpus), "steps": args.steps,
                          "warmup": args.warmup,
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
    # per-step CUDA events on torch's stream: each library call returns with its result
    # complete (it synchronises its own stream), so the events bracket whole factorizations
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    results = []
    with ClockSampler(local_rank) as clk:
        barrier()
        evs[0].record()
        for i in range(args.steps):
            r = one_step()
            evs[i + 1].record()
            results.append((r.timing, r.rank, [len(a) for a in r.accepted], r.relative_trace_error))
            r.free()
        barrier()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    t = torch.tensor([sum(step_ms), statistics.median(step_ms)], device=dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, median_ms = float(t[0].item()), float(t[1].item())
    sec_per_step = median_ms / 1e3
    timing, k_final, m_seq, trace_err = results[-1]
    upd_ms = timing["update_ms"]
    flops = timing["update_flops"]
    peak, peak_src = fp64_peak()
    # rounds whose residual GEMM ran on the tensor cores (int8 digit planes): their time and
    # the FP64 flops they replaced are split out, so each kernel is held to its own roof
    tc_ms, tc_ops, tc_fl = timing["tc_ms"], timing["tc_int8_ops"], timing["tc_fp64_flops"]
    fp64_ms, fp64_flops = upd_ms - tc_ms, flops - tc_fl
    achieved = fp64_flops / (fp64_ms * 1e-3) / 1e12 if fp64_ms > 0 else 0.0
    tr = ncu_traffic(w.name + ("_lowmem" if lowmem else "") + ("_tc" if tc_ms > 0 else ""))
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

    # same-run parity on the full workload; the oracle run is also the CPU baseline
    cpu, parity = None, None
    if rank == 0 and world == 1 and not lowmem and not args.no_parity:
        parity, t_cpu = same_run_parity(w, x, spec, cfg, ctx, x_dev, n_cores)
        if not args.no_cpu:
            cpu = {"value": t_cpu, "unit": "s", "cores": n_cores, "kind": "port",
                   "cpu_model": cpu_model(),
                   "sample": f"full {w.name} workload (N={w.n}, no extrapolation): the C "
                             f"restatement of the reference (oracle/rpc_oracle.c, OpenMP over "
                             f"rows, {n_cores} threads), the same run that checks parity"}
    elif rank == 0 and world == 1 and not args.no_cpu:
        n_sample = args.cpu_sample or min(w.n, 10_000 if lowmem else 100_000)
        dt, ext = cpu_sample(w, n_cores, n_sample, lowmem)
        cpu = {"value": ext, "unit": "s", "cores": n_cores, "kind": "port",
               "cpu_model": cpu_model(),
               "sample": f"oracle restatement on the first N'={n_sample} rows of {w.name}, same "
                         f"k/b/seed, {dt:.2f} s measured, x N/N' to the full N"}

    if rank == 0:
        roof_fp64 = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": ("lowmem_kernel (A(R, S_all) regenerated in SMEM + FP64 DMMA GEMM "
                                "with the new L^-1 rows + diag update)") if lowmem else
                               ("update_kernel (fused kernel columns + L^-T + diag update; the "
                                "residual GEMM on FP64 DMMA in the rounds below RPC_I8_MIN_K, "
                                "added from the tensor-core launch above it)"),
                     "traffic_note": traffic_note,
                     "note": ("rounds whose residual GEMM runs on the int8 tensor cores leave this "
                              "kernel the Gram, the kernel-function transform, A L^-T and the "
                              "epilogue (ncu round 9: DMMA 47 % + FP64 19 % of the shared FP64 "
                              "pipe, profiles/r02_update_kernel_ncu_r9_s4.txt); the whole update "
                              "step is in update_step.frac_of_fp64_peak") if tc_ms > 0 else None,
                     "peak_source": peak_src,
                     "per_launch_flops": fp64_flops / max(1, timing["update_launches"]),
                     "kernel_ms_per_step": fp64_ms,
                     "share_of_step": fp64_ms / (sec_per_step * 1e3)}
        roof_tc = None
        if tc_ms > 0:
            i8_peak, i8_src = int8_peak()
            tc_ach = tc_ops / (tc_ms * 1e-3) / 1e12
            roof_tc = {"bound": "tensor", "achieved": tc_ach, "peak": i8_peak, "unit": "TOP/s (int8)",
                       "frac": tc_ach / i8_peak if i8_peak else None, "traffic": None,
                       "kernel": ("i8gemm2_kernel (residual GEMM F B'^T from 7 int8 digit planes per "
                                  "operand, tcgen05.mma kind::i8 M=128 N=m, int32 TMEM accumulators, "
                                  "two passes over K: diagonals 0-3 then 4-6; i8gemm_kernel for m <= 64)"),
                       "peak_source": i8_src,
                       "fp64_equivalent_tflops": tc_fl / (tc_ms * 1e-3) / 1e12,
                       "kernel_ms_per_step": tc_ms,
                       "digit_plane_append_ms_per_step": timing["tc_slice_ms"],
                       "share_of_step": tc_ms / (sec_per_step * 1e3)}
        # the dominant kernel carries "roofline"
        roof_main = roof_fp64
        if roof_tc is not None and tc_ms > fp64_ms:
            roof_main, roof_tc = roof_tc, roof_fp64
        line = {
            "metric": METRIC, "value": sec_per_step, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "step_ms": {"median": median_ms, "mean": total_ms / args.steps,
                        "min": min(step_ms), "max": max(step_ms)},
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads.py)", "config": cfg_json,
            "kernel_col_gbs": col_gbs,
            "rank_final": k_final, "rounds": len(m_seq), "accepted_per_round": m_seq,
            "relative_trace_error": trace_err,
            "device_factorize_ms": timing["factorize_ms"],
            "host_ms": {k: round(timing[k], 3) for k in ("host_total_ms", "host_setup_ms",
                                                         "host_loop_ms", "host_final_ms",
                                                         "upload_ms")},
            "roofline": roof_main,
            "roofline_secondary": roof_tc,
            "update_step": {"ms": upd_ms, "fp64_flops": flops,
                            "fp64_equivalent_tflops": flops / (upd_ms * 1e-3) / 1e12 if upd_ms else None,
                            # the whole update step (int8 residual GEMM + fused FP64 kernel + digit
                            # appends) against the FP64 DMMA peak the round-1 design was bound by
                            "frac_of_fp64_peak": (flops / (upd_ms * 1e-3) / 1e12 / peak)
                            if (upd_ms and peak) else None,
                            "share_of_step": upd_ms / (sec_per_step * 1e3)},
            "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
            "gpu_launches": int(timing["kernel_launches"]) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
