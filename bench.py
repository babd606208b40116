#!/usr/bin/env python
"""Benchmark of the KPM moment engine (BASELINE.json metric: D*N*R vector-element
updates/s and HBM GB/s at 1/2/4/8 B200).

One "step" = one whole kpm_moments call = the full hot path on
one batch: generate the R random vectors, first step, floor(N/2)-1 fused recursion steps,
fixed-order finish, (N > 1 ranks: the library's one NCCL all-reduce of the sums), doubling
assembly.  Default workload: BASELINE.json configs[3] (2D Peierls lattice 1024x1024,
complex128, N=4096, R=256), the largest configuration that fits one GPU's share of the work
(configs[4] is the row-partitioned multi-GPU case, `--config c5 --partition rows`).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
                  [--scaling strong|weak]

--gpus N > 1 without torchrun's environment re-launches this script under
`python -m torch.distributed.run --nproc-per-node N` (one process per GPU).  Ranks own the
global vectors kpm_vector_range(R, rank, N): strong scaling by default
(the config's R split over the ranks), --scaling weak keeps R per GPU.  With as many GPUs as
ranks the library owns the collective (KPM_COMM_NCCL: one ncclAllReduce of the moment sums
inside kpm_moments); with fewer GPUs than ranks (tests) ranks share GPUs and the raw sums go
through one gloo all-reduce.  Rank 0 prints ONE JSON line on stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
UNIT = "updates/s"
L2_BYTES = 126e6
_OUT = sys.stdout  # replaced in main() by the saved stdout descriptor


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


def kernel_name(fmt, plan):
    if fmt == "csr":
        return "kpm_ell_step_kernel (ELL SpMM over the vector block + recursion + reductions)"
    if fmt == "dense":
        return "kpm_dense_step_kernel (DMMA fp64 GEMM H~ a_n + fused recursion and moment sums)"
    if plan.get("four_step"):
        return "kpm_step_quad_kernel (four recursion steps per HBM pass, TMA-fed march)"
    if plan.get("three_step"):
        return "kpm_step_tri_kernel (three recursion steps per HBM pass, TMA-fed march)"
    if plan.get("ks"):
        return f"kpm_stepk_tma_kernel ({plan['ks']} recursion steps per launch)"
    if plan.get("two_step"):
        return "kpm_step2_tma_kernel (two recursion steps per HBM pass, TMA-fed march)"
    if plan.get("box3"):
        return "kpm_step3_tma_kernel (3D TMA march, dense halo box per plane)"
    if plan.get("tma"):
        return "kpm_step_tma_kernel (TMA-fed march)"
    return "kpm_step_kernel (fused stencil SpMM + recursion + reductions)"


def profiled_traffic(config, kname, R_loc, fmt):
    """dram__bytes_read.sum + dram__bytes_write.sum per step launch from the committed ncu
    capture of this config's step kernel at this R per GPU (profiles/traffic.json), or None."""
    try:
        recs = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return None, None
    key = config if fmt in (None, "stencil") else f"{config}_{fmt}"
    rec = recs.get(f"{key}_R{R_loc}") or recs.get(key)
    if not rec or rec.get("R_loc") != R_loc:
        return None, None  # no capture of this config at this R per GPU
    if kname.split(" ")[0] not in rec.get("kernel", ""):
        return None, None  # the committed capture is of another kernel: no traffic claim
    return rec["dram_bytes_per_launch"], rec.get("round")


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


class OracleSampler:
    """The oracle as it stands (oracle/kpm_oracle.c, OpenMP), on a bounded sample of the workload:
    full D, R' vectors (one per host thread, more when the whole N fits the budget), the first
    N' <= N moments, sized once by a short calibration so that one sample takes ~target_s.
    value = D*N'*R'/s of the sample."""

    def __init__(self, cfg, lat, a, b, target_s, dense=False):
        # every host core (torchrun sets OMP_NUM_THREADS=1 for its workers; the oracle's OpenMP
        # runtime reads the variable when liboracle.so is first loaded)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
        import oracle
        self.oracle = oracle
        self.H = oracle.csr_from_dense(ki.lattice_dense(lat), keep_zeros=True) if dense else oracle.lattice_csr(lat)
        self.a, self.b, self.cfg, self.D = a, b, cfg, lat["D"]
        threads = oracle.num_threads()
        self.threads = threads
        # one vector per thread (fewer vectors than threads: the oracle splits rows instead); huge D:
        # at most 4 vectors (the oracle keeps 3 full vectors per vector in flight)
        Rs = min(cfg["R"], threads if self.D <= (1 << 24) else 4)
        r = ki.rademacher(cfg["seed"], Rs, self.D)
        t0 = time.perf_counter()
        oracle.moments_doubling(self.H, a, b, r, 4)            # 2 products per vector
        t4 = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.moments_doubling(self.H, a, b, r, 12)           # 6 products per vector
        per_product = max((time.perf_counter() - t0 - t4) / 4, t4 / 8, 1e-9)
        Ns = int(min(cfg["N"], max(4, 2 * int(target_s / per_product))))
        reps = 1
        if Ns == cfg["N"]:  # the whole N fits: widen to more vectors, then repeat the whole workload
            est = per_product * Ns / 2
            Rs = int(min(cfg["R"], Rs * max(1, int(target_s / max(est, 1e-9)))))
            est *= Rs / min(cfg["R"], threads)
            if Rs == cfg["R"]:
                reps = int(max(1, min(100000, target_s / max(est, 1e-9))))
        self.Rs, self.Ns, self.reps = Rs, Ns, reps
        self.r = ki.rademacher(cfg["seed"], Rs, self.D)

    def run(self):
        import oracle  # noqa: F401  (already loaded)
        t0 = time.perf_counter()
        for _ in range(self.reps):
            self.oracle.moments_doubling(self.H, self.a, self.b, self.r, self.Ns)
        dt = time.perf_counter() - t0
        return self.D * self.Ns * self.Rs * self.reps / dt, dt

    def describe(self, dt):
        cores = self.threads
        rep = f", whole workload x{self.reps}" if self.reps > 1 else ""
        return (f"{self.Rs} of {self.cfg['R']} vectors (global 0..{self.Rs - 1}), full D={self.D}, first {self.Ns} "
                f"of N={self.cfg['N']} moments ({self.Ns // 2} products per vector){rep}; {dt:.2f} s wall on "
                f"{cores} OpenMP threads of {self.threads}; CSR build excluded"), cores


def config_obj(args, cfg, lat, world, R_total, R_loc, fmt, l2_resident):
    rows = args.partition == "rows"
    wl = (f"BASELINE.json configs[{int(args.config[1]) - 1}]: {cfg['name']}" if args.config.startswith("c")
          else cfg["name"])
    return {"workload": wl, "config": args.config,
            "D": lat["D"], "N": cfg["N"], "R_total": R_total, "R_per_gpu": R_loc, "ndim": lat["ndim"],
            "L": list(lat["L"]), "t": lat["t"], "anderson_W": cfg["W"], "flux": lat["flux"],
            "vector_seed": cfg["seed"], "disorder_seed": cfg["disorder_seed"],
            "parallelism": f"rows{world}" if rows else f"vectors{world}",
            "H_format": fmt,
            "l2": ("L2-resident vector blocks (2 x D*R*s < 126 MB L2): not an HBM number" if l2_resident
                   else "inputs larger than L2 (2 x D*R*s vector blocks > 126 MB), no flush needed")}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n):
    """--gpus N > 1 outside torchrun: one process per GPU through torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    rc = subprocess.call(cmd, stdout=_OUT, stderr=sys.stderr)
    sys.exit(rc)


def run_reference(args, cfg, lat, rank, world):
    """The reference arm of this tier: the oracle as it stands on the host cores, rank 0 only,
    each step a bounded sample of the workload sized so the whole run ends in a few minutes."""
    if rank != 0:
        return
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    import oracle
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    target = min(15.0, max(2.0, 120.0 / max(1, args.steps + args.warmup)))
    sm = OracleSampler(cfg, lat, a, b, target, dense=args.format == "dense")
    steps = []
    for i in range(args.warmup + args.steps):
        v, dt = sm.run()
        if i >= args.warmup:
            steps.append((v, dt))
    value = statistics.median(v for v, _ in steps)
    sample, cores = sm.describe(statistics.median(d for _, d in steps))
    R_total = cfg["R"] * (world if args.scaling == "weak" else 1)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(d for _, d in steps),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "c128" if lat["flux"] else "f64", "data": "synthetic",
            "config": config_obj(args, cfg, lat, world, R_total, R_total, args.format,
                                 2 * lat["D"] * R_total * (16 if lat["flux"] else 8) < L2_BYTES),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=_OUT, flush=True)


def main():
    # stdout carries exactly one JSON line: libraries that print to fd 1 (NCCL's version banner)
    # are sent to stderr; the result line is written to the saved descriptor.
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(ki.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's R split over the ranks (SURVEY 8(e) E = T1/(G TG)); "
                         "weak: R vectors per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--format", default=None, choices=["stencil", "csr", "dense"],
                    help="how H reaches the library: lattice-stencil descriptor, the same H as CSR "
                         "(kpm_create_csr -> ELL; general sparse path), or dense (the paper's own variant; "
                         "default for config pd)")
    ap.add_argument("--dist-backend", default="auto", choices=["auto", "nccl", "gloo"],
                    help="auto: NCCL (the library's communicator) when every rank has its own GPU, else gloo "
                         "(ranks share GPUs; the raw sums go through one gloo all-reduce)")
    ap.add_argument("--r-per-gpu", type=int, default=None,
                    help="override the vectors per GPU (R_total = this x ranks), e.g. c2 with 8: one GPU's "
                         "share of c2 at 8 GPUs under strong scaling")
    ap.add_argument("--partition", default="vectors", choices=["vectors", "rows"],
                    help="vectors: SURVEY 8(e) P1; rows: slabs of the slowest dimension with halo exchange "
                         "every step (P2, BASELINE.json configs[4])")
    ap.add_argument("--halo", default="ipc", choices=["ipc", "nccl"],
                    help="row partition: ipc = KPM_COMM_IPC, the recursion kernels store boundary planes straight "
                         "into the neighbours' ghost planes (CUDA IPC / NVLink peer memory, fused halo); nccl = "
                         "KPM_COMM_NCCL send/recv of the planes overlapped with the interior")
    ap.add_argument("--plan", default="", help="kpm_plan_opts for A/B runs, e.g. 'no_two_step=1,tma_lanes=8'")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(ki.CONFIGS[args.config])
    lat = ki.lattice(cfg)
    if args.format is None:
        args.format = cfg.get("format", "stencil")
    rows = args.partition == "rows"
    if args.r_per_gpu:
        cfg["R"] = args.r_per_gpu * (1 if rows else world)
        args.scaling = "strong"
    R_total = cfg["R"] * (world if (args.scaling == "weak" and not rows) else 1)

    if args.impl == "reference":
        run_reference(args, dict(cfg, R=R_total), lat, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1105_5481_b200 import kpm
    ndev = max(torch.cuda.device_count(), 1)
    shared = world > ndev  # more ranks than GPUs (multi-rank tests on one GPU)
    backend = args.dist_backend if args.dist_backend != "auto" else ("gloo" if shared else "nccl")
    local_rank = local_rank % ndev
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    lib_comm = world > 1 and backend == "nccl"

    a, b = kpm.kpm_gershgorin_stencil(lat["ndim"], lat["L"], lat["t"], onsite=lat["onsite"], flux=lat["flux"])
    N = cfg["N"]
    if rows or args.format != "stencil":
        args.no_e2e = True  # (e2e below re-creates a stencil handle)
    if rows:
        if args.halo == "ipc":
            name = [kpm.kpm_ipc_unique_name() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(name, src=0)
            part = (kpm.KPM_PART_ROWS, rank, world, kpm.KPM_COMM_IPC, name[0])
        else:
            if world == 1:
                dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % free_port(), rank=0, world_size=1)
            part = (kpm.KPM_PART_ROWS, rank, world, kpm.KPM_COMM_NCCL, kpm.nccl_id_for_group())
        R_loc = R_total
    elif world > 1:
        part = ((kpm.KPM_PART_VECTORS, rank, world, kpm.KPM_COMM_NCCL, kpm.nccl_id_for_group()) if lib_comm
                else (kpm.KPM_PART_VECTORS, rank, world))
        R_loc = kpm.kpm_vector_range(R_total, rank, world)[1]
    else:
        part, R_loc = None, R_total
    Hd = None
    if args.format == "csr":
        assert not rows, "the row partition is benchmarked for stencils"
        rowptr, col, val = ki.lattice_csr(lat)
        a, b = kpm.kpm_gershgorin_csr(lat["D"], rowptr, col, val)
        h = kpm.kpm_create_csr(lat["D"], rowptr, col, val, a, b, device=local_rank, dist=part)
    elif args.format == "dense":
        assert not rows, "the row partition is benchmarked for stencils"
        Hd = ki.lattice_dense(lat)
        a, b = kpm.kpm_gershgorin_dense(Hd)
        h = kpm.kpm_create_dense(Hd, a, b, device=local_rank, dist=part)
    else:
        h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                   device=local_rank, dist=part)
    if args.plan:
        h.set_plan_opts(**{k: int(v) for k, v in (kv.split("=") for kv in args.plan.split(","))})
    stream = torch.cuda.Stream(device=dev)
    h.set_stream(stream.cuda_stream)
    ws_bytes = h.workspace_size(N, R_total)
    ws = torch.empty(ws_bytes + 256, dtype=torch.uint8, device=dev)
    h.set_workspace((ws.data_ptr() + 255) // 256 * 256, ws_bytes)
    S = torch.empty(N, dtype=torch.float64, device=dev)
    mu = torch.empty(N, dtype=torch.float64, device=dev)

    def step():
        if rows or lib_comm or world == 1:
            # the whole call inside the library: recursion, (the NCCL all-reduce of the sums), assembly
            h.moments_ex(N, R_total, cfg["seed"], flags=kpm.KPM_DEVICE_OUT, out=mu.data_ptr())
            return
        # ranks sharing a GPU: raw sums, one gloo all-reduce through host memory, device assembly
        h.moments_ex(N, R_total, cfg["seed"], flags=kpm.KPM_RAW_SUMS | kpm.KPM_DEVICE_OUT, out=S.data_ptr())
        stream.synchronize()
        Sh = S.cpu()
        dist.all_reduce(Sh)
        S.copy_(Sh)
        h.assemble(S.data_ptr(), N, R_total, out=mu.data_ptr())

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    steps_ms, step_launches, launches, alg_bytes, design_bytes = 0.0, 0, 0, 0.0, 0.0
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            ms, sl, tl = h.last_timing()   # events the library records around its step launches
            ab, db = h.step_traffic()      # SURVEY 8(d) algorithmic / compulsory DRAM bytes of those launches
            steps_ms += ms
            step_launches += sl
            alg_bytes += ab
            design_bytes += db
            launches += tl + (0 if (rows or lib_comm or world == 1) else 1)
        ev1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize(dev)
    barrier()
    ms_total = ev0.elapsed_time(ev1)
    rdev = dev if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([ms_total], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    D = lat["D"]
    value = D * N * R_total / (ms_per_step / 1000.0)
    mu_host = mu.cpu().numpy()
    s_el = 16 if lat["flux"] else 8
    l2_resident = 2 * D * R_loc * s_el < L2_BYTES

    # end to end through the public API with host buffers, per step: kpm_create_stencil (H2D of
    # H~'s data from pinned host memory: on-site energies / Peierls phases), kpm_moments (random
    # vectors drawn on the GPU as the paper does; mu D2H to the host), kpm_destroy.
    e2e = None
    if not args.no_e2e:
        onsite_bytes = 0 if lat["onsite"] is None else lat["onsite"].nbytes
        phase_bytes = 16 * lat["L"][0] if lat["flux"] else 0
        pinned_onsite = None
        if lat["onsite"] is not None:
            pinned_onsite = torch.from_numpy(lat["onsite"]).pin_memory().numpy()

        def e2e_step():
            h2 = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=pinned_onsite,
                                        flux=lat["flux"], device=local_rank, dist=part)
            if world > 1 and not lib_comm:
                out = kpm.moments_distributed(h2, N, R_total, cfg["seed"], device=torch.device("cpu"))
            else:
                out = h2.moments(N, R_total, cfg["seed"])  # (KPM_COMM_NCCL: the shared communicator)
            h2.close()
            return out
        e2e_step()
        k = max(1, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_out = e2e_step()
        e2e_ms = (time.perf_counter() - t0) * 1000 / k
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=rdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item())
        assert np.array_equal(e2e_out, mu_host), "e2e result differs from the device-resident run"
        e2e = {"value": D * N * R_total / (e2e_ms / 1000.0), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(onsite_bytes + phase_bytes + 64), "d2h_bytes_per_step": 8 * N,
               "path": "kpm_create_stencil + kpm_moments (host mu) + kpm_destroy per step, wall clock, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sm = OracleSampler(dict(cfg, R=R_total), lat, a, b, 15.0, dense=Hd is not None)
        v, dt = sm.run()
        sample, cores = sm.describe(dt)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}

    plan = h.plan_info(N, R_total) if args.format != "dense" else {"dense": 1, "tile": "64x64x32 DMMA m8n8k4"}
    kname = kernel_name(args.format, plan)
    avg_launch_ms = steps_ms / max(step_launches, 1)
    peak, peak_kind = peak_hbm()
    if Hd is None:
        achieved = alg_bytes / (steps_ms / 1000.0) / 1e9
        traffic, traffic_round = profiled_traffic(args.config, kname, R_loc, args.format)
        roofline = {
            "bound": "hbm", "kernel": kname,
            # 3 D R s (+ 8 D on-site, + ELL bytes) per recursion step, whatever the kernel;
            # a two-step launch (temporal blocking) counts two steps but moves ~2/3 of their bytes
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": (f"profiles/traffic.json ({traffic_round}, ncu dram__bytes_read.sum"
                                                   " + dram__bytes_write.sum per steady-state launch)"
                                                   if traffic else None),
            "alg_bytes_per_launch": alg_bytes / max(step_launches, 1),
            "design_bytes_per_launch": design_bytes / max(step_launches, 1),
            "design_gbs": design_bytes / (steps_ms / 1000.0) / 1e9,
            "dram_gbs": traffic / (avg_launch_ms / 1000.0) / 1e9 if traffic else None,
            "dram_frac": traffic / (avg_launch_ms / 1000.0) / 1e9 / peak if traffic else None,
            "avg_launch_ms": avg_launch_ms, "launches_per_step": step_launches / args.steps,
            "frac_of_8TBs_spec": achieved / 8000.0, "l2_resident": l2_resident, "plan": plan}
    else:
        # a dense fp64 contraction: algorithmic flops 2 D^2 R per recursion step (unpadded) over the
        # step launches' device time, against cuBLAS DGEMM measured here on the same shape
        flops = 2.0 * D ** 2 * R_loc * step_launches
        achieved_tf = flops / (steps_ms / 1000.0) / 1e12
        peak_tf = measure_dgemm_tflops(dev, D, R_loc)
        roofline = {"bound": "tensor", "kernel": kname, "achieved": achieved_tf, "peak": peak_tf,
                    "peak_kind": "measured (torch.matmul float64 = cuBLAS DGEMM, same M, N, K, in this run)",
                    "unit": "TFLOP/s", "frac": achieved_tf / peak_tf, "traffic": None,
                    "alg_flops_per_launch": 2.0 * D ** 2 * R_loc, "avg_launch_ms": avg_launch_ms,
                    "frac_of_40TF_spec": achieved_tf / 40.0, "plan": plan}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if (rows or args.scaling == "strong") else "weak",
                "vs_baseline": None, "dtype": "c128" if lat["flux"] else "f64",
                "data": "synthetic (seeded Rademacher vectors generated on the GPU, lattice H of the config)",
                "config": config_obj(args, cfg, lat, world, R_total, R_loc, args.format, l2_resident),
                "collective": (("KPM_COMM_IPC: fused peer-plane halo stores in the recursion kernels, interprocess "
                                "event ordering, rank-order sum of the moment sums over mapped workspaces")
                               if rows and args.halo == "ipc" else
                               ("library NCCL all-reduce of the moment sums (KPM_COMM_NCCL)" if (lib_comm or rows)
                                else ("gloo all-reduce of raw sums (ranks share GPUs)" if world > 1 else None))),
                "devices": min(world, ndev),
                # the whole job's algorithmic bytes over the step time
                "hbm_gbs_alg": alg_bytes / args.steps * world / (ms_per_step / 1000.0) / 1e9,
                # the metric counts D*N*R (two moments per product with doubling);
                # the products actually performed are floor(N/2) per vector
                "physical_updates_per_s": D * (N // 2) * R_total / (ms_per_step / 1000.0),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "halo_stats": h.last_stats() if rows else None,
                "clocks": clk.summary(), "mu_check": {"mu0": float(mu_host[0]),
                                                        "max_abs_mu": float(np.abs(mu_host).max())}}
        print(json.dumps(line), file=_OUT, flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
