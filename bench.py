#!/usr/bin/env python
"""Benchmark of the KPM moment engine (BASELINE.json metric: D*N*R vector-element
updates/s and HBM GB/s).

One "step" = one whole kpm_moments call = the full hot path on one batch: generate
R random vectors, first step, floor(N/2)-1 fused recursion steps, fixed-order
finish, doubling assembly (and, for N > 1 ranks, the one all-reduce of the sums).
Default workload: BASELINE.json configs[1] (2D square lattice 512x512, N=1024,
R=64, fp64), whose vector block (2 x 134 MB) exceeds the 126 MB L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
Under torchrun each rank owns R vectors of its own (random-vector partition,
weak scaling); rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import kpm_inputs as ki  # noqa: E402

METRIC = "KPM vector-element updates/s (D*N*R/s)"
_OUT = sys.stdout  # replaced in main() by the saved stdout descriptor
UNIT = "updates/s"


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic(config, plan):
    """dram__bytes_read.sum + dram__bytes_write.sum per step launch from the committed ncu
    capture of this config's step kernel (profiles/*.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        rec = json.load(open(p))[config]
    except Exception:
        return None
    want = ("stepk" if plan.get("ks") else "step2" if plan.get("two_step")
            else "step3_tma" if plan.get("box3") else ("step_tma" if plan.get("tma") else "kpm_step_kernel"))
    if want not in rec.get("kernel", ""):
        return None  # the committed capture is of another kernel: no traffic claim
    return rec["dram_bytes_per_launch"]


def measure_dgemm_tflops(dev, D, R, reps=10):
    """fp64 tensor-core reference: cuBLAS DGEMM (torch.matmul on float64) of the dense step's
    shape (D x D) x (D x R), CUDA events, after warm-up."""
    import torch
    A = torch.randn(D, D, dtype=torch.float64, device=dev)
    B = torch.randn(D, R, dtype=torch.float64, device=dev)
    C = torch.matmul(A, B)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(A, B, out=C)
    e1.record()
    torch.cuda.synchronize(dev)
    return 2.0 * D * D * R * reps / (e0.elapsed_time(e1) / 1000.0) / 1e12


def oracle_sample(cfg, lat, a, b, target_s=15.0, dense=False):
    """The oracle as it stands, on a bounded sample of the workload: full D, R' vectors
    (one per host thread, fewer for huge D; more, up to R, when all N moments take well under
    target_s), and the first N' <= N moments chosen from a short calibration run so the sample
    takes ~target_s.  Returns D*N'*R'/s.  dense: H is
    handed to the oracle with all D^2 entries (the dense variant's arithmetic)."""
    import oracle
    H = oracle.csr_from_dense(ki.lattice_dense(lat), keep_zeros=True) if dense else oracle.lattice_csr(lat)
    threads = oracle.num_threads()
    D = lat["D"]
    Rs = min(cfg["R"], threads if D <= (1 << 24) else max(1, min(threads, 4)))
    r = ki.rademacher(cfg["seed"], Rs, D)
    t0 = time.perf_counter()
    oracle.moments_doubling(H, a, b, r, 4)                    # 2 products per vector
    t4 = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.moments_doubling(H, a, b, r, 12)                   # 6 products per vector
    per_product = max((time.perf_counter() - t0 - t4) / 4, t4 / 8)
    Ns = int(min(cfg["N"], max(4, 2 * int(target_s / max(per_product, 1e-9)))))
    t0 = time.perf_counter()
    oracle.moments_doubling(H, a, b, r, Ns)
    dt = time.perf_counter() - t0
    if Ns == cfg["N"] and dt < target_s / 3 and Rs < cfg["R"]:  # all N moments fit: widen to more vectors
        Rs = int(min(cfg["R"], Rs * max(1, int(target_s / max(dt, 1e-9)))))
        r = ki.rademacher(cfg["seed"], Rs, D)
        t0 = time.perf_counter()
        oracle.moments_doubling(H, a, b, r, Ns)
        dt = time.perf_counter() - t0
    reps = 1
    for _ in range(3):  # the whole workload is small: repeat it until the sample is long enough
        if not (Ns == cfg["N"] and Rs == cfg["R"] and dt < target_s / 3) or reps >= 100000:
            break
        reps = int(min(100000, reps * max(2, target_s / max(dt, 1e-6))))
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.moments_doubling(H, a, b, r, Ns)
        dt = time.perf_counter() - t0
    value = D * Ns * Rs * reps / dt
    cores = min(threads, Rs)
    sample = (f"{Rs} of {cfg['R']} vectors (global 0..{Rs - 1}), full D={D}, first {Ns} of N={cfg['N']} moments "
              f"({Ns // 2} products per vector){f", whole workload x{reps}" if reps > 1 else ""}; {dt:.2f} s wall on {cores} OpenMP threads; CSR build excluded")
    return value, cores, sample, dt


def run_reference(args, cfg, lat, a, b, rank, world):
    if rank != 0:
        return
    steps = []
    for i in range(args.warmup + args.steps):
        v, threads, sample, dt = oracle_sample(cfg, lat, a, b)
        if i >= args.warmup:
            steps.append((v, dt))
    value = statistics.median(v for v, _ in steps)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(d for _, d in steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_obj(args, cfg, lat, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=_OUT, flush=True)


def config_obj(args, cfg, lat, world):
    rows = getattr(args, "partition", "vectors") == "rows"
    wl = (f"BASELINE.json configs[{int(args.config[1]) - 1}]: {cfg['name']}" if args.config.startswith("c")
          else cfg["name"])
    return {"workload": wl, "config": args.config,
            "D": lat["D"], "N": cfg["N"], "R_per_gpu": cfg["R"] if not rows else None,
            "R_total": cfg["R"] * (1 if rows else world), "ndim": lat["ndim"],
            "L": list(lat["L"]), "t": lat["t"], "anderson_W": cfg["W"], "flux": lat["flux"],
            "vector_seed": cfg["seed"], "disorder_seed": cfg["disorder_seed"],
            "parallelism": f"rows{world}" if rows else f"vectors{world}",
            "H_format": getattr(args, "format", "stencil"),
            "l2": ("inputs larger than L2 (2 x D*R*s vector blocks)"
                   if 2 * lat["D"] * cfg["R"] * (16 if lat["flux"] else 8) > 126e6
                   else "L2-resident vector blocks (2 x D*R*s < 126 MB L2): not an HBM number")}


def main():
    # stdout carries exactly one JSON line: libraries that print to fd 1 (NCCL's version banner)
    # are sent to stderr; the result line is written to the saved descriptor.
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(ki.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--format", default=None, choices=["stencil", "csr", "dense"],
                    help="how H reaches the library: lattice-stencil descriptor, the same H as CSR "
                         "(kpm_create_csr -> ELL; general sparse path), or dense (the paper's own variant; "
                         "default for config pd)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: all-reduce through host memory; lets several "
                         "ranks share one GPU to test the multi-rank path)")
    ap.add_argument("--r-per-gpu", type=int, default=None,
                    help="override the config's vectors per GPU (e.g. c2 with R=8: one GPU's share of c2 "
                         "at 8 GPUs under strong scaling, whose vector blocks stay in L2)")
    ap.add_argument("--partition", default="vectors", choices=["vectors", "rows"],
                    help="vectors: each rank owns R vectors of its own (weak scaling, one all-reduce); rows: "
                         "the lattice is cut into slabs of the slowest dimension with halo exchange over NCCL "
                         "every step (strong scaling, BASELINE.json configs[4])")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = ki.CONFIGS[args.config]
    if args.r_per_gpu:
        cfg = dict(cfg, R=args.r_per_gpu)
    lat = ki.lattice(cfg)
    if args.format is None:
        args.format = cfg.get("format", "stencil")

    if args.impl == "reference":
        import oracle
        a, b = oracle.gershgorin(oracle.lattice_csr(lat))
        run_reference(args, cfg, lat, a, b, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1105_5481_b200 import kpm
    local_rank = local_rank % max(torch.cuda.device_count(), 1)  # several ranks may share a GPU (gloo tests)
    torch.cuda.set_device(local_rank)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local_rank)

    a, b = kpm.kpm_gershgorin_stencil(lat["ndim"], lat["L"], lat["t"], onsite=lat["onsite"], flux=lat["flux"])
    N, R_loc = cfg["N"], cfg["R"]
    rows = args.partition == "rows"
    if rows or args.format == "csr":
        args.no_e2e = True  # (e2e below re-creates a stencil or dense handle)
    if rows:
        if world == 1:
            dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % (29500 + os.getpid() % 1000),
                                    rank=0, world_size=1)
        R = R_loc
        part = (kpm.KPM_PART_ROWS, rank, world, kpm.KPM_COMM_NCCL, kpm.nccl_id_for_group())
    else:
        R = R_loc * world
        part = (kpm.KPM_PART_VECTORS, rank, world)
    Hd = None
    if args.format == "csr":
        assert not rows, "the row partition is implemented for stencils"
        rowptr, col, val = ki.lattice_csr(lat)
        a, b = kpm.kpm_gershgorin_csr(lat["D"], rowptr, col, val)
        h = kpm.kpm_create_csr(lat["D"], rowptr, col, val, a, b, device=local_rank, dist=part)
    elif args.format == "dense":
        assert not rows, "the row partition is implemented for stencils"
        Hd = ki.lattice_dense(lat)
        a, b = kpm.kpm_gershgorin_dense(Hd)
        h = kpm.kpm_create_dense(Hd, a, b, device=local_rank, dist=part)
    else:
        h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                   device=local_rank, dist=part)
    stream = torch.cuda.Stream(device=dev)
    h.set_stream(stream.cuda_stream)
    ws_bytes = h.workspace_size(N, R)
    ws = torch.empty(ws_bytes + 256, dtype=torch.uint8, device=dev)
    base = (ws.data_ptr() + 255) // 256 * 256
    h.set_workspace(base, ws_bytes)
    S = torch.empty(N, dtype=torch.float64, device=dev)
    mu = torch.empty(N, dtype=torch.float64, device=dev)

    def step():
        if rows:  # halo exchange and the moment all-reduce run inside the library (NCCL)
            mu.copy_(torch.from_numpy(h.moments(N, R, cfg["seed"])))
            return
        h.moments_ex(N, R, cfg["seed"], flags=kpm.KPM_RAW_SUMS | kpm.KPM_DEVICE_OUT, out=S.data_ptr())
        if world > 1:
            if args.dist_backend == "nccl":
                with torch.cuda.stream(stream):
                    dist.all_reduce(S)  # the one collective of the vector partition (NCCL, NVLink)
            else:
                stream.synchronize()
                Sh = S.cpu()
                dist.all_reduce(Sh)
                S.copy_(Sh)
        h.assemble(S.data_ptr(), N, R, out=mu.data_ptr())

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    steps_ms, step_launches, launches, steps_bytes = 0.0, 0, 0, 0.0
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            ms, sl, tl = h.last_timing()   # events the library records on its stream
            steps_ms += ms
            step_launches += sl
            steps_bytes += h.step_bytes()  # algorithmic bytes of those step launches
            launches += tl + 1             # + the assemble kernel
        ev1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize(dev)
    ms_total = ev0.elapsed_time(ev1)
    rdev = dev if (world == 1 or args.dist_backend == "nccl") else torch.device("cpu")
    t = torch.tensor([ms_total], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_per_step = float(t.item()) / args.steps
    D = lat["D"]
    value = D * N * R / (ms_per_step / 1000.0)

    # roofline of the dominant kernel: the fused recursion step
    peak, peak_kind = peak_hbm()
    plan = h.plan_info(N, R) if args.format != "dense" else {"dense": 1, "tile": "64x64x32 DMMA m8n8k4"}
    kname = ("kpm_ell_step_kernel (ELL SpMM over the vector block, cp.async-staged row entries, + recursion + "
             "reductions; kpm_step_kernel<EllOp> for K > 16 or KPM_ELL_GENERIC)"
             if args.format == "csr" else
             "kpm_dense_step_kernel (DMMA fp64 GEMM H~ a_n + fused recursion and moment sums)"
             if args.format == "dense" else
             f"kpm_stepk_tma_kernel ({plan['ks']} recursion steps per HBM pass, TMA-fed march; remainder steps "
             "by the two-/single-step kernels, included)" if plan.get("ks")
             else "kpm_step2_tma_kernel (two recursion steps per HBM pass, TMA-fed march)" if plan.get("two_step")
             else "kpm_step3_tma_kernel (3D TMA march, dense halo box per plane, z rolled in registers; fused "
                  "stencil SpMM + recursion + reductions)" if plan.get("box3")
             else "kpm_step_tma_kernel (TMA-fed march: fused stencil SpMM + recursion + reductions)" if plan.get("tma")
             else "kpm_step_kernel (fused stencil SpMM + recursion + reductions)")
    avg_step_ms = steps_ms / max(step_launches, 1)
    step_bytes = steps_bytes / max(step_launches, 1)
    achieved = steps_bytes / (steps_ms / 1000.0) / 1e9
    mu_host = mu.cpu().numpy()

    # end-to-end through the public API with host buffers: create (H2D of H~'s data),
    # moments (random vectors drawn on the GPU, as the paper does), D2H of mu.
    e2e = None
    if not args.no_e2e:
        onsite_bytes = 0 if lat["onsite"] is None else lat["onsite"].nbytes
        phase_bytes = 16 * lat["L"][0] if lat["flux"] else 0
        pinned_onsite = None
        if lat["onsite"] is not None:
            pinned_onsite = torch.from_numpy(lat["onsite"]).pin_memory().numpy()

        if Hd is not None:
            Hd_pinned = torch.from_numpy(Hd).pin_memory().numpy()
            onsite_bytes, phase_bytes = Hd.nbytes, 0

        def e2e_step():
            if Hd is not None:
                h2 = kpm.kpm_create_dense(Hd_pinned, a, b, device=local_rank, dist=part)
            else:
                h2 = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=pinned_onsite,
                                            flux=lat["flux"], device=local_rank, dist=part)
            if world > 1:
                out = kpm.moments_distributed(h2, N, R, cfg["seed"],
                                              device=None if args.dist_backend == "nccl" else torch.device("cpu"))
            else:
                out = h2.moments(N, R, cfg["seed"])
            h2.close()
            return out
        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 5))):
            e2e_out = e2e_step()
        k = max(1, min(args.steps, 5))
        e2e_ms = (time.perf_counter() - t0) * 1000 / k
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=rdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item())
        assert np.array_equal(e2e_out, mu_host), "e2e result differs from the device-resident run"
        e2e = {"value": D * N * R / (e2e_ms / 1000.0), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(onsite_bytes + phase_bytes + 64), "d2h_bytes_per_step": 8 * N,
               "path": ("kpm_create_dense" if Hd is not None else "kpm_create_stencil") +
                       " + kpm_moments (host mu) + kpm_destroy per step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, threads, sample, _ = oracle_sample(cfg, lat, a, b, dense=Hd is not None)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample}

    if Hd is None:
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": profiled_traffic(args.config, plan),
                    "alg_bytes_per_launch": step_bytes, "avg_launch_ms": avg_step_ms,
                    "frac_of_8TBs_spec": achieved / 8000.0, "plan": plan}
    else:
        # a dense fp64 contraction: algorithmic flops 2 D^2 R per recursion step (unpadded) over the
        # step launches' device time, against cuBLAS DGEMM measured here on the same shape
        flops = 2.0 * lat["D"] ** 2 * R_loc * step_launches
        achieved_tf = flops / (steps_ms / 1000.0) / 1e12
        peak_tf = measure_dgemm_tflops(dev, lat["D"], R_loc)
        roofline = {"bound": "tensor", "kernel": kname, "achieved": achieved_tf, "peak": peak_tf,
                    "peak_kind": "measured (torch.matmul float64 = cuBLAS DGEMM, same M, N, K, in this run)",
                    "unit": "TFLOP/s", "frac": achieved_tf / peak_tf, "traffic": None,
                    "alg_flops_per_launch": 2.0 * lat["D"] ** 2 * R_loc, "avg_launch_ms": avg_step_ms,
                    "frac_of_40TF_spec": achieved_tf / 40.0, "plan": plan}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if rows else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Rademacher vectors, lattice H)",
                "config": config_obj(args, cfg, lat, world),
                "hbm_gbs_alg": steps_bytes / args.steps / (ms_per_step / 1000.0) / 1e9 * world,
                # the metric counts D*N*R (two moments per product with doubling);
                # the products actually performed are floor(N/2) per vector
                "physical_updates_per_s": lat["D"] * (cfg["N"] // 2) * R
                / (ms_per_step / 1000.0),
                "roofline": roofline,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "mu_check": {"mu0": float(mu_host[0]),
                                                        "max_abs_mu": float(np.abs(mu_host).max())}}
        print(json.dumps(line), file=_OUT, flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
