"""S^3CMTF SGD epoch benchmark (BASELINE.json metric: tensor+matrix nonzero SGD
updates/sec per epoch; % roofline).

Workload at N=1 (default): BASELINE configs[4] ("config5") at its largest
point, the largest single-GPU configuration: a 1e7 x 1e7 x 1e7 tensor with
1e9 uniform nonzeros (90/10 split -> 9e8 training entries), planted core
10^3 + N(0, 0.1) noise, coupled 1e7 x 1e6 matrix on mode 1 with 1e8
nonzeros; rank 10, S^3CMTF-opt.  Synthetic, seeded, generated on the device.
Other configs are behind --config (config2 = configs[1], config3 =
configs[2], config4 = configs[3]; config5 --nnz/--rank for the sweep points).

A "step" = one run_epoch (tensor sweep + matrix sweeps + non-finite scan)
over the device-resident bundle.  `value` = updates/s on the device (CUDA
events on the launching stream); `e2e` = the same through the C ABI with
host buffers (bundle upload + epoch + stats read back each step).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

With --gpus N > 1 outside torchrun, the script launches itself under
torch.distributed.run (one process per GPU) so the DSGD path runs.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP32_FMA_PER_SM_CLK = 128  # Blackwell SM: 4 x 32 FP32 lanes
# arithmetic type of each epoch kernel (the parameters and accumulators are
# fp32 everywhere; the tcgen05 kernel forms its products from split fp16
# operands, hi*hi + hi*lo + lo*hi, ~22 mantissa bits -- fp32-level accuracy)
DTYPE = {"order3tm": "f32 (tcgen05 MMAs on split-fp16 x3 operands, fp32 accumulate)",
         "order3v2": "f32 (core gradient: tf32 mma.sync)",
         "order4": "f32 (mma.sync on split 3xTF32 operands, fp32 accumulate)",
         "order4tm": "f32 (tcgen05 MMAs on split-fp16 x3 operands, fp32 accumulate)",
         "order3": "f32", "generic": "f32"}
CONFIG_INDEX = {"config1": "BASELINE configs[0]", "config2": "BASELINE configs[1]",
                "config3": "BASELINE configs[2]", "config4": "BASELINE configs[3]",
                "config5": "BASELINE configs[4]"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="config5")
    p.add_argument("--scale", type=float, default=1.0)
    p.add_argument("--nnz", type=float, default=1e9, help="config5 tensor nonzeros")
    p.add_argument("--rank", type=int, default=10, help="config5 rank")
    p.add_argument("--kernel", default="opt", choices=["opt", "naive"])
    p.add_argument("--hog-threads", type=int, default=0)
    p.add_argument("--order", default="random", choices=["sorted", "random"])
    p.add_argument("--uniform", action="store_true",
                   help="diagnostic: uniform instead of Zipf indices")
    p.add_argument("--cpu-sample", type=int, default=1_000_000,
                   help="tensor entries in the bounded CPU-baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-naive", action="store_true")
    p.add_argument("--strong", action="store_true",
                   help="DSGD (N > 1): fixed total workload instead of weak scaling")
    p.add_argument("--dsgd", action="store_true",
                   help="use the DSGD/NCCL path even with one rank (testing)")
    return p.parse_args()


def physical_cores():
    """Physical cores counted the way the reference's acceptance test does
    (tests/acceptance.cpp:52-73): distinct (physical id, core id) pairs in
    /proc/cpuinfo, else the hardware concurrency."""
    ids, phys, core = set(), -1, -1
    try:
        with open("/proc/cpuinfo") as f:
            for line in list(f) + [""]:
                line = line.rstrip("\n")
                if not line:
                    if core >= 0:
                        ids.add((0 if phys < 0 else phys, core))
                    phys = core = -1
                elif line.startswith("physical id"):
                    phys = int(line.split(":", 1)[1])
                elif line.startswith("core id"):
                    core = int(line.split(":", 1)[1])
    except OSError:
        pass
    return len(ids) if ids else (os.cpu_count() or 1)


def relaunch_under_torchrun(args):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N processes (one per GPU) and return its exit
    code, so the DSGD path engages whichever way the driver launches us."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def make_workload(args, mult=1.0, device_gen=False):
    """The BASELINE workload; `mult` scales its size (multi-GPU weak scaling,
    generated on the device)."""
    from paper_1708_08640_b200 import synth
    if args.config == "config2" and device_gen:
        from paper_1708_08640_b200 import synth_gpu
        spec = synth_gpu.config2(args.scale * mult)
        bundle, test = synth_gpu.generate(spec, device=f"cuda:{dist_env()[2]}")
        return spec, bundle, test, [10, 10, 10], 1e-3, 0.01
    if args.config == "config2":
        spec = synth.config2(args.scale)
        if args.uniform:
            spec.laws = ["uniform"] * 3
            for m in spec.matrices:
                m.row_law = m.col_law = "uniform"
        ranks = [10, 10, 10]
        lr, lam = 1e-3, 0.01
    elif args.config == "config1":
        spec = synth.config1(literal=False)
        ranks, lr, lam = [5, 5, 5], 0.01, 0.01
    elif args.config in ("config3", "config4", "config5"):
        # device-side generation (1e8 - 1e9 nonzeros)
        from paper_1708_08640_b200 import synth_gpu
        if args.config == "config3":
            spec = synth_gpu.config3(args.scale * mult)
        elif args.config == "config4":
            spec = synth_gpu.config4(args.scale * mult)
        else:
            spec = synth_gpu.config5(args.nnz * mult, args.rank)
        bundle, test = synth_gpu.generate(spec, device=f"cuda:{dist_env()[2]}")
        return spec, bundle, test, list(spec.ranks), 1e-3, 0.01
    else:
        raise SystemExit(f"unknown config {args.config}")
    bundle, test, _ = synth.generate(spec)
    return spec, bundle, test, ranks, lr, lam


def host_bundle(bundle, lo=0, hi=None):
    """Host (numpy) view of a possibly device-resident bundle (prefix sample)."""
    from paper_1708_08640_b200.api import DataBundle
    if hasattr(bundle.tensor, "to_host"):
        t = bundle.tensor.to_host(lo, hi)
        frac = (t.nnz / bundle.tensor.nnz) if bundle.tensor.nnz else 1.0
        return DataBundle(t, [m.to_host(0, int(m.nnz * frac)) for m in bundle.matrices])
    return bundle


def algorithmic(bundle, ranks):
    """B_t = 8N+4+8 sum J, F_t = 6 prod J; B_m = 16+16J, F_m = 10J."""
    N = len(ranks)
    nt = bundle.tensor.nnz
    Bt, Ft = 8 * N + 4 + 8 * sum(ranks), 6 * int(np.prod(ranks))
    mats = [(m.nnz, ranks[m.coupled_mode]) for m in bundle.matrices]
    return nt, Bt, Ft, mats


class ClockSampler:
    """SM clocks and throttle reasons DURING the timed region: NVML polled
    every 5 ms from a background thread (nvidia-smi -lms cannot sample a
    tens-of-milliseconds window densely enough)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
                    time.sleep(0.005)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception:
            self._t = None

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(1)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "NVML, 5 ms polling"}


def cpu_baseline(bundle, ranks, lr, lam, sample, steps=2, warmup=1, threads=None,
                 kernel_opt=True):
    """The reference's own multi-threaded run_epoch (oracle/_ref) on a bounded
    sample of the workload: the first `sample` training entries plus the same
    fraction of every coupled matrix, workers = physical cores."""
    from oracle import oracle as O
    from paper_1708_08640_b200.api import CoupledMatrix, DataBundle, SparseTensor
    bundle = host_bundle(bundle, 0, min(sample, bundle.tensor.nnz))
    t = bundle.tensor
    frac = min(1.0, sample / t.nnz)
    st = SparseTensor(t.dims, t.indices[:sample], t.values[:sample])
    ms = [CoupledMatrix(m.coupled_mode, m.rows, m.cols, m.indices[: int(m.nnz * frac)],
                        m.values[: int(m.nnz * frac)], m.weight) for m in bundle.matrices]
    sb = DataBundle(st, ms)
    cores = threads or physical_cores()
    run = O.RefRun(sb, ranks, seed=0, eta0=lr, mu=0.1, lambda_reg=lam, workers=cores,
                   kernel_opt=kernel_opt)
    for _ in range(warmup):
        run.run_epoch()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run.run_epoch()
        times.append(time.perf_counter() - t0)
    run.close()
    n_upd = st.nnz + sum(m.nnz for m in ms)
    return n_upd / min(times), n_upd, cores, times


def sample_text(n_sample, nt, nsamp, cores, kernel):
    return (f"first {n_sample} of {nt} training entries ({100.0 * n_sample / max(1, nt):.3g}%) "
            f"+ the same fraction of each matrix ({nsamp} updates per epoch); the reference's "
            f"run_epoch (oracle/_ref, kernel {kernel}) with workers = {cores} physical cores, "
            "best of the timed epochs after 1 warm-up")


def fp32_peak_tflops(sms, mhz):
    return sms * FP32_FMA_PER_SM_CLK * 2 * mhz * 1e6 / 1e12


def workload_name(args):
    return (f"{args.config} ({CONFIG_INDEX.get(args.config, '?')})"
            + (f", nnz {args.nnz:g}, rank {args.rank}" if args.config == "config5"
               else f", scale {args.scale:g}"))


def run_reference(args):
    """The reference arm: the reference's own CPU run_epoch (oracle/_ref, the
    unmodified sources compiled here) with all physical cores, on a bounded
    sample of the same workload (each step = one epoch over the sample).
    Rank 0 alone runs under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    spec, bundle, test, ranks, lr, lam = make_workload(args)
    nt = bundle.tensor.nnz
    n_sample = min(args.cpu_sample, nt)
    ups, n_upd, cores, times = cpu_baseline(bundle, ranks, lr, lam, args.cpu_sample,
                                            steps=max(1, args.steps), warmup=args.warmup)
    nups, _, _, ntimes = cpu_baseline(bundle, ranks, lr, lam, args.cpu_sample, steps=1,
                                      warmup=0, kernel_opt=False)
    line = {
        "metric": "tensor+matrix nonzero SGD updates/sec per epoch", "impl": "reference",
        "value": ups, "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * min(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args) + f" -- bounded sample: {n_sample} of {nt} "
                               "training entries per step",
                   "sample_tensor_entries": n_sample, "updates_per_step": n_upd,
                   "ranks": ranks, "kernel": "opt"},
        "cpu_baseline": {"value": ups, "unit": "updates/s", "cores": cores,
                         "kind": "reference",
                         "sample": sample_text(n_sample, nt, n_upd, cores, "opt"),
                         "naive": {"value": nups, "unit": "updates/s",
                                   "ms_per_step": 1e3 * min(ntimes)}},
        "e2e": {"value": ups, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    from paper_1708_08640_b200 import api
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    spec, bundle, test, ranks, lr, lam = make_workload(args)
    cfg = api.TrainConfig(ranks=ranks, seed=rank, eta0=lr, lambda_reg=lam, kernel=args.kernel,
                          device=local, hog_threads=args.hog_threads,
                          order_policy=args.order,
                          core_flush_every=int(os.environ.get("CMTF_BENCH_CORE_EVERY", "0")))
    st = api.make_state(cfg, bundle)
    nt, Bt, Ft, mats = algorithmic(bundle, ranks)
    n_upd = nt + sum(n for n, _ in mats)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    for _ in range(args.warmup):
        api.run_epoch(st)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    per = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed epochs (inputs are also > L2)
        torch.cuda.synchronize()
        api.run_epoch(st)
        per.append(st.last_epoch_timing())
    torch.cuda.synchronize()
    clk = clocks.stop()
    tot_ms = sum(p["total_ms"] for p in per)
    ten_ms = sum(p["tensor_ms"] for p in per) / len(per)
    mat_ms = sum(p["matrix_ms"] for p in per) / len(per)
    ms_step = tot_ms / len(per)
    if world > 1:
        t = torch.tensor([ms_step], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_step = float(t.item())
    value = n_upd * world / (ms_step * 1e-3)
    info = st.kernel_info()
    launches = sum(p["launches"] for p in per)
    stats = api.epoch_stats(st, lam)
    test_rmse = api.test_rmse(st, test)

    # roofline of the dominant kernel (tensor sweep): FP32 flops / its event time
    props = torch.cuda.get_device_properties(local)
    sms = props.multi_processor_count
    peak_nominal = fp32_peak_tflops(sms, 1965.0)
    # the binding bound is the slower of the gather bytes at
    # HBM bandwidth and the flops at FP32 peak (J = 10: FP32; J = 5: HBM)
    hbm_peak = 6548.5e9
    hbm_src = "fallback 6548.5 GB/s"
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        pass
    bytes_t = nt * Bt
    hbm_bound = Bt / hbm_peak > Ft / (peak_nominal * 1e12)
    if hbm_bound:
        achieved = bytes_t / (ten_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak / 1e9, "unit": "GB/s",
                "frac": achieved / (hbm_peak / 1e9), "traffic": None, "peak_source": hbm_src}
    else:
        achieved = nt * Ft / (ten_ms * 1e-3) / 1e12
        roof = {"bound": "fp32", "achieved": achieved, "peak": peak_nominal, "unit": "TFLOP/s",
                "frac": achieved / peak_nominal, "traffic": None,
                "peak_source": f"nominal FP32: {sms} SMs x 128 FMA x 2 x 1965 MHz (no FP32 "
                               "entry in MEASURED_PEAKS.json)"}
    # the factor rows of the large configs are random 48-byte rows in tables
    # far beyond L2: the memory system's measured ceiling for that access
    # pattern (scripts/micro/red_bench.cu on this B200: ~1.8e10 random row
    # gathers/s, ~1.3-1.9e10 random row updates/s) bounds the sweep before
    # either term above does
    rows_per_s = (len(ranks) * nt + 2 * sum(n for n, _ in mats)) / (ten_ms * 1e-3)
    roof.update({
            "kernel": {"order3v2": "hog3v2_kernel (fused tensor+matrix epoch sweep)",
                       "order3tm": "hog3tm_kernel (fused epoch sweep, tcgen05 contractions + "
                                   "core gradient, TMEM accumulators)",
                       "order4": "hog4_kernel (fused epoch sweep, tensor-core contractions)",
                       "order4tm": "hog4tm_kernel (fused epoch sweep, tcgen05 contractions + core "
                                   "gradient, TMEM accumulators)",
                       "order3": "hog3_kernel (tensor sweep)",
                       "generic": "hogwild_generic_kernel (tensor sweep)"}.get(info["kernel"]),
            "kernel_ms": ten_ms,
            "flops_per_update": Ft, "bytes_per_update": Bt,
            "gather_gbs": bytes_t / (ten_ms * 1e-3) / 1e9,
            "fp32_tflops": nt * Ft / (ten_ms * 1e-3) / 1e12,
            "row_updates_per_s": rows_per_s,
            "random_row_ceiling_per_s": 1.8e10,
            "frac_at_measured_clock": ((nt * Ft / (ten_ms * 1e-3) / 1e12)
                                       / fp32_peak_tflops(sms, clk["sm_mhz"])
                                       if clk.get("sm_mhz") and not hbm_bound else None)})
    if info["kernel"] in ("order3tm", "order4tm"):
        roof["note"] = ("flops are the algorithmic 6*prod(J) per update of SURVEY 8(d), counted "
                        "against the CUDA-core FP32 peak; the tcgen05 kernels run the "
                        "contractions on the tensor cores (three fp16 MMAs per product, fp32 "
                        "accumulate) and ~3J^2 (order 3) / ~5J^2 (order 4) FP32 FMAs per update, "
                        "so the fraction is not capped by 1")
    # DRAM traffic per launch of the dominant kernel, from the committed ncu
    # --set full capture of the same command (profiles/ncu_r1_metrics.json)
    try:
        prof = {}
        for fn in ("ncu_r1_metrics.json", "ncu_r2_metrics.json"):  # later rounds override
            fp = os.path.join(ROOT, "profiles", fn)
            if os.path.exists(fp):
                prof.update(json.load(open(fp)))
        key = {"order3v2": "hog3v2", "order3tm": "hog3tm", "order4": "hog4",
               "order4tm": "hog4tm"}.get(info["kernel"])
        for k, v in prof.items():
            # keys: "<kernel> <config> [scale s | nnz n rank j] (...)"
            if args.config == "config5":
                want = f"nnz {args.nnz:g} rank {args.rank}"
                scale_ok = want in k
            else:
                scale_ok = (f"scale {args.scale:g}" in k) if "scale" in k else args.scale == 1.0
            if key and k.startswith(key) and args.config in k.replace("(", " ").split() and scale_ok:
                roof["traffic"] = (v["dram__bytes_read.sum"]["value"]
                                   + v["dram__bytes_write.sum"]["value"]) * 1e6
                roof["traffic_unit"] = "bytes/launch (ncu dram read+write)"
                roof["traffic_source"] = v["report"]
                roof["algorithmic_bytes_per_launch"] = nt * Bt
                pick = {"fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                        "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                        "ipc": "sm__inst_executed.avg.per_cycle_active",
                        "instructions": "smsp__inst_executed.sum"}
                roof["ncu"] = {kk: v[name]["value"] for kk, name in pick.items() if name in v}
    except Exception:
        pass
    # epoch roofline time: both terms, slower of HBM and FP32
    hbm = hbm_peak
    t_roof = nt * max(Bt / hbm, Ft / (peak_nominal * 1e12)) + sum(
        n * max((16 + 16 * j) / hbm, 10 * j / (peak_nominal * 1e12)) for n, j in mats)
    roof["epoch_roofline_frac"] = t_roof / (ms_step * 1e-3)

    line = {
        "metric": "tensor+matrix nonzero SGD updates/sec per epoch", "value": value,
        "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE.get(info["kernel"], "f32"), "data": "synthetic",
        "config": {"workload": workload_name(args),
                   "tensor_entries": nt, "matrix_entries": [n for n, _ in mats],
                   "ranks": ranks, "kernel": args.kernel, "lr": lr, "lambda": lam,
                   "hog_threads": info["hog_threads"], "tensor_kernel": info["kernel"],
                   "sort_mode": info["sort_mode"], "l2": "flushed between epochs (256 MiB "
                   f"write); the COO records ({nt * 16 / 1e6:.0f} MB) also exceed L2",
                   "parallelism": f"dp{world}" if world > 1 else "single"},
        "breakdown_ms": {"tensor": ten_ms, "matrix": mat_ms,
                         "scan": sum(p["scan_ms"] for p in per) / len(per)},
        "quality": {"train_rmse": stats.train_rmse, "test_rmse": test_rmse,
                    "epochs_done": st.epoch},
        "roofline": roof, "clocks": clk, "gpu_launches": launches,
    }

    if not args.no_e2e:
        # e2e through the C ABI with host buffers: upload the bundle, run the
        # epoch, read the stats back, every step (wall clock).
        h2d = bundle.tensor.indices.nbytes + bundle.tensor.values.nbytes + sum(
            m.indices.nbytes + m.values.nbytes for m in bundle.matrices)
        # the caller's host buffers live in pinned memory (as a data loader's would),
        # first touched from the GPU-local CPUs (what `numactl --cpunodebind` gives a
        # job on a multi-socket host; a no-op on this pool's single-node 16-vCPU VMs,
        # whose upload rate still varied between 18 and 46 GB/s from run to run --
        # `upload_gbs` says what this run got)
        from paper_1708_08640_b200.api import CoupledMatrix, DataBundle, SparseTensor
        aff0, numa = None, "unbound"
        try:
            import pynvml
            pynvml.nvmlInit()
            aff0 = os.sched_getaffinity(0)
            pr = torch.cuda.get_device_properties(local)
            hnd = pynvml.nvmlDeviceGetHandleByPciBusId(
                f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
            words = pynvml.nvmlDeviceGetCpuAffinity(hnd, (os.cpu_count() + 63) // 64)
            cpus = {64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1}
            cpus &= aff0
            if cpus:
                os.sched_setaffinity(0, cpus)
                numa = f"host buffers pinned from the GPU-local CPUs ({len(cpus)} of {len(aff0)})"
        except Exception as ex:  # no NVML / not permitted: stay unbound
            numa = f"unbound ({type(ex).__name__})"

        def pinned(a):
            if hasattr(a, "data_ptr"):  # device tensor: pinned host copy
                return a.cpu().pin_memory()
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t.numpy()

        t = bundle.tensor
        if hasattr(t, "to_host"):
            from paper_1708_08640_b200.synth_gpu import DeviceBundle, DeviceMatrix, DeviceTensor
            pb = DeviceBundle(DeviceTensor(t.dims, pinned(t.indices), pinned(t.values)),
                              [DeviceMatrix(m.coupled_mode, m.rows, m.cols, pinned(m.indices),
                                            pinned(m.values), m.weight)
                               for m in bundle.matrices])
            h2d = pb.tensor.indices.nbytes + pb.tensor.values.nbytes + sum(
                m.indices.nbytes + m.values.nbytes for m in pb.matrices)
            bundle = pb
        else:
            pb = DataBundle(SparseTensor(t.dims, pinned(t.indices), pinned(t.values)),
                            [CoupledMatrix(m.coupled_mode, m.rows, m.cols, pinned(m.indices),
                                           pinned(m.values), m.weight)
                             for m in bundle.matrices])
            bundle = pb
        # the device-generated copies are no longer needed (the context holds
        # its own records): free them before re-uploading from the host
        st.bundle = bundle
        del t, pb
        test = None
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        if aff0 is not None:  # pinned pages are placed: give the threads back
            os.sched_setaffinity(0, aff0)
        ts, parts = [], []
        for k in range(max(2, args.steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st.upload(bundle)
            t1 = time.perf_counter()
            api.run_epoch(st)
            t2 = time.perf_counter()
            s = api.epoch_stats(st, lam)
            t3 = time.perf_counter()
            ts.append(t3 - t0)
            parts.append((t1 - t0, t2 - t1, t3 - t2))
        e2e_s = statistics.median(ts)
        med = [1e3 * statistics.median(p[i] for p in parts) for i in range(3)]
        line["e2e"] = {"value": n_upd * world / e2e_s, "unit": "updates/s",
                       "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 16,
                       "ms_per_step": 1e3 * e2e_s,
                       "breakdown_ms": {"upload": med[0], "epoch": med[1], "stats": med[2]},
                       "includes": "set_tensor+add_matrix (H2D, validate, sort), run_epoch, "
                                   "epoch_stats",
                       "upload_gbs": h2d / (med[0] * 1e-3) / 1e9, "numa": numa}
    if rank == 0 and not args.no_cpu_baseline:
        n_sample = min(args.cpu_sample, nt)
        ups, nsamp, cores, times = cpu_baseline(bundle, ranks, lr, lam, args.cpu_sample)
        line["cpu_baseline"] = {"value": ups, "unit": "updates/s", "cores": cores,
                                "kind": "reference",
                                "sample": sample_text(n_sample, nt, nsamp, cores, "opt")}
    if not args.no_naive and args.kernel == "opt":
        # S^3CMTF-naive beside opt (BASELINE configs[1]: "naive vs cached-opt"),
        # same bundle, a fresh state
        st.close()
        del st
        torch.cuda.empty_cache()
        cfgn = api.TrainConfig(ranks=ranks, seed=rank, eta0=lr, lambda_reg=lam, kernel="naive",
                               device=local, hog_threads=args.hog_threads,
                               order_policy=args.order)
        stn = api.make_state(cfgn, bundle)
        api.run_epoch(stn)
        pn = []
        for _ in range(2):
            flush.zero_()
            torch.cuda.synchronize()
            api.run_epoch(stn)
            pn.append(stn.last_epoch_timing())
        ms_n = sum(p["total_ms"] for p in pn) / len(pn)
        line["naive"] = {"value": n_upd * world / (ms_n * 1e-3), "unit": "updates/s",
                         "ms_per_step": ms_n, "tensor_kernel": stn.kernel_info()["kernel"],
                         "steps": 2, "warmup": 1}
        stn.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_dsgd(args):
    """N > 1: DSGD over the ranks (one process per GPU).
    Every rank generates the workload on its own device (same seed), keeps
    only its own entries (device partition, dsgd.partition_rank), and runs
    the stratified epoch: stratum sweeps, ring rotation of the stratified
    row blocks (ncclSend / ncclRecv) and delta all-reduces of the replicated
    parameters, all on the context's stream.  Config 5 stratifies all three
    1e7-row modes (G^2 steps); the others modes 1 and 2.  BASELINE's
    multi-GPU configs (3 - 5) keep the total workload fixed (strong scaling);
    config 2 grows with N (weak scaling: config 2 at N x its nonzeros, every
    GPU a config-2-sized share) unless --strong."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1708_08640_b200 import api, dsgd
    from paper_1708_08640_b200.synth_gpu import DeviceBundle, DeviceMatrix, DeviceTensor
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"), rank=rank,
                            world_size=world)
    n_strat = 3 if args.config == "config5" else 2
    weak = not args.strong and args.config in ("config1", "config2")
    spec, bundle, test, ranks, lr, lam = make_workload(
        args, mult=world if weak else 1.0, device_gen=True)
    dev = f"cuda:{local}"
    if not hasattr(bundle.tensor, "to_host"):  # host-generated (config 1): to the device
        t = bundle.tensor
        bundle = DeviceBundle(
            DeviceTensor(t.dims, torch.from_numpy(t.indices.view(np.int32)).to(dev),
                         torch.from_numpy(t.values).to(dev)),
            [DeviceMatrix(m.coupled_mode, m.rows, m.cols,
                          torch.from_numpy(m.indices.view(np.int32)).to(dev),
                          torch.from_numpy(m.values).to(dev), m.weight) for m in bundle.matrices])
    nt, Bt, Ft, mats = algorithmic(bundle, ranks)
    n_upd = nt + sum(n for n, _ in mats)
    plan, counts, col_counts, nnz = dsgd.partition_rank(bundle, world, rank, n_strat=n_strat)
    del bundle
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    cfg = api.TrainConfig(ranks=ranks, seed=0, eta0=lr, lambda_reg=lam, kernel=args.kernel,
                          device=local)
    rs = dsgd.RankState(plan, rank, cfg, counts, col_counts, nnz)
    obj = [dsgd.new_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    dsgd.comm_init(rs, world, rank, obj[0])
    L, h = rs.state._L, rs.state._h
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        dsgd.run_epoch_nccl(rs)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    per = []
    ms = C.c_double()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        rs.state._check(L.cmtf_gpu_mark(h, 0))
        dsgd.run_epoch_nccl(rs)
        rs.state._check(L.cmtf_gpu_mark(h, 1))
        rs.state._check(L.cmtf_gpu_elapsed_ms(h, 0, 1, C.byref(ms)))
        per.append(ms.value)
    clk = clocks.stop()
    t = torch.tensor([sum(per) / len(per)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    value = n_upd / (ms_step * 1e-3)
    props = torch.cuda.get_device_properties(local)
    peak = fp32_peak_tflops(props.multi_processor_count, 1965.0) * world
    achieved = nt * Ft / (ms_step * 1e-3) / 1e12
    sch = plan.schedule
    n_rot = sum(len(sch.rotations_after(s)) for s in range(sch.steps))
    n_sync = bin(plan.shared_modes).count("1") + bin(plan.mat_mask).count("1") + 1
    launches = args.steps * (sch.steps * (1 + 2 * n_sync) + 2 + len(ranks) + len(mats))
    # quality: consolidate the blocks, test RMSE on the held-out split;
    # train RMSE from every rank's local SSE
    dsgd.consolidate_nccl(rs)
    torch.cuda.synchronize()
    st_local = api.epoch_stats(rs.state, lam)
    sse = torch.tensor([st_local.train_rmse ** 2 * plan.bundle.tensor.nnz], device=dev,
                       dtype=torch.float64)
    dist.all_reduce(sse)
    train_rmse = float((sse / nnz).sqrt().item())
    test_rmse = api.test_rmse(rs.state, test) if rank == 0 else None
    # e2e: re-upload the rank's local bundle from pinned host memory, run the
    # epoch, read the stats back (wall clock, max over ranks)
    lb = plan.bundle
    pb = DeviceBundle(DeviceTensor(lb.tensor.dims, lb.tensor.indices.cpu().pin_memory(),
                                   lb.tensor.values.cpu().pin_memory()),
                      [DeviceMatrix(m.coupled_mode, m.rows, m.cols, m.indices.cpu().pin_memory(),
                                    m.values.cpu().pin_memory(), m.weight) for m in lb.matrices])
    h2d = pb.tensor.indices.nbytes + pb.tensor.values.nbytes + sum(
        m.indices.nbytes + m.values.nbytes for m in pb.matrices)
    rs.plan.bundle = pb
    rs.state.bundle = pb
    del lb, test
    gc.collect()
    torch.cuda.empty_cache()
    ts = []
    for _ in range(max(2, min(args.steps, 3))):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        rs.reupload()
        dsgd.run_epoch_nccl(rs)
        api.epoch_stats(rs.state, lam)
        ts.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.median(ts)], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    hb = torch.tensor([float(h2d)], device=dev, dtype=torch.float64)
    dist.all_reduce(hb)
    if rank == 0:
        line = {
            "metric": "tensor+matrix nonzero SGD updates/sec per epoch", "value": value,
            "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if weak else "strong",
            "vs_baseline": None, "dtype": "f32 (tcgen05 MMAs on split-fp16 x3 operands, "
                                          "fp32 accumulate)", "data": "synthetic",
            "config": {"workload": workload_name(args)
                       + (f", x{world} (weak scaling: one config-sized share per GPU, "
                          "device-generated)" if weak else ", fixed total (strong scaling)"),
                       "tensor_entries": nt, "matrix_entries": [n for n, _ in mats],
                       "ranks": ranks, "kernel": args.kernel, "lr": lr, "lambda": lam,
                       "parallelism": f"dsgd{world}: {n_strat}-mode strata, {sch.steps} steps "
                                      "per epoch, row blocks rotated with ncclSend/ncclRecv, "
                                      "replicated deltas all-reduced per step",
                       "l2": "flushed between epochs"},
            "quality": {"train_rmse": train_rmse, "test_rmse": test_rmse,
                        "epochs_done": rs.state.epoch},
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "peak_source": f"nominal FP32 x {world} GPUs",
                         "kernel": "whole DSGD epoch (sweeps + NCCL rotations / reductions)"},
            "clocks": clk, "gpu_launches": launches, "rotations_per_epoch": n_rot,
            "e2e": {"value": n_upd / float(te.item()), "unit": "updates/s",
                    "h2d_bytes_per_step": int(hb.item()), "d2h_bytes_per_step": 16 * world,
                    "ms_per_step": 1e3 * float(te.item())},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[1] > 1 or args.dsgd:
        run_dsgd(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
