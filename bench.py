#!/usr/bin/env python
"""Benchmark of the FFT tensor-sketch hot path (BASELINE.json metric:
"tensor-sketch build entries/s (HBM GB/s) and sketched T(I,u,u) contractions/s").

Headline workload (N=1 and every N): BASELINE config 2, the largest single-GPU dense
config -- a symmetric n=1000 fp32 tensor (1e9 entries, 4 GB), rank-100 planted + 0.01
mirrored Gaussian noise, generated on the device from a seed; symmetric sketch b=2^16,
B=10. One step = one full sketch build over the sorted triples (sketch.cpp:315-345) of
the tensor resident in HBM; with N ranks the i-slices are split by equal work and the
B x b sketches are summed with an NCCL all-reduce (strong scaling). `value` = n^3
logical entries per second for the whole job. Extra keys: the config-1 build (n=400
fp64, b=2^14, B=20) and the sketched-contraction throughput (batched T(I,u,u) over L=100
restarts, the RTPM power step) on that sketch.

--impl reference times the reference algorithm's CPU implementation (the oracle
restatement in oracle/ -- the reference itself needs Eigen3/FFTW3, absent here) on the
host cores, rank 0 only, over a bounded i-slice sample of the same config-2 workload.
That arm builds its input with the oracle's own generator and never loads the product
library.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tensor-sketch build entries/s (HBM GB/s) and sketched T(I,u,u) contractions/s"
CFG = dict(n=1000, rank=100, sigma=0.01, b=1 << 16, B=10, seed=20150615)  # config 2 (fp32)
CFG1 = dict(n=400, rank=50, sigma=0.01, b=1 << 14, B=20, seed=20150615, L=100)  # config 1 (fp64)
REF_ROWS = 40  # CPU sample: rows i in [0, 40) of config 2 = 11.5% of the sorted triples
PRODUCT_LIB = "libsketchcp_b200.so"


def simplex_entries(n, i0=0, i1=None):
    i1 = n if i1 is None else i1
    return sum((n - i) * (n - i + 1) // 2 for i in range(i0, i1))


def equal_work_slices(n, world):
    """Contiguous i-ranges with about equal sorted-triple counts (distributed.equal_work_slices,
    restated so this module imports without the product library)."""
    tot = simplex_entries(n)
    bounds, acc, r = [0], 0, 1
    for i in range(n):
        acc += (n - i) * (n - i + 1) // 2
        while r < world and acc >= tot * r / world:
            bounds.append(i + 1)
            r += 1
    while len(bounds) < world:
        bounds.append(n)
    bounds.append(n)
    return [(bounds[k], bounds[k + 1]) for k in range(world)]


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region.

    NVML (pynvml) is queried every ~1 ms from a side thread, so even a ~20 ms timed region
    gets a median over many samples; nvidia-smi (~50 ms per query) is the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, device, interval=0.001):
        self.device = device
        self.interval = interval
        self.rows = []
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._h = None
            try:  # the CUDA ordinal may differ from NVML's index: match by PCI bus id
                import torch

                pr = torch.cuda.get_device_properties(int(device))
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(int(device))
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.rows.append([str(sm), str(self._max), hex(rs)] + ["Active" if rs & bit else "Not Active" for bit in self.BITS])

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            self.rows.append([x.strip() for x in out.stdout.strip().split(",")])

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self._sample_nvml()
                    self.source = "nvml"
                else:
                    self._sample_smi()
                    self.source = "nvidia-smi"
            except Exception:
                self._nvml = None  # fall back to nvidia-smi for the rest of the region
            self._stop.wait(self.interval if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.rows:  # region shorter than one query: take one right after it
            try:
                self._sample_nvml() if self._nvml is not None else self._sample_smi()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_min_mhz": min(sm) if sm else None, "reasons": reasons, "samples": len(self.rows),
                "source": self.source}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(kernel, config):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        e = d.get(f"{kernel}@{config}") or d.get(kernel)
        if e and e.get("config") == config:
            return e.get("dram_bytes_per_launch")
    return None


def pcie_link(device):
    """Current / max PCIe generation and width of the GPU's link (the e2e leg is bus-bound)."""
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(device), "--query-gpu=pcie.link.gen.current,pcie.link.gen.max,"
                              "pcie.link.width.current,pcie.link.width.max", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5)
        g, gm, w, wm = [x.strip() for x in out.stdout.strip().split(",")]
        return {"gen": g, "gen_max": gm, "width": w, "width_max": wm}
    except Exception:
        return None


def _microbench_rows():
    for name in ("r02_atomics.jsonl", "r01_microbench_atomics.jsonl"):
        p = ROOT / "profiles" / name
        if p.exists():
            rows = [json.loads(l) for l in p.read_text().splitlines() if l.strip().startswith("{")]
            return rows, f"profiles/{name}"
    return None, None


def scatter_roofline(adds, kernel_ms, limbs=2, gather_stride=None):
    """The ceilings the scatter actually meets, from the microbenchmarks
    (microbench/atomics.cu): (1) the exact adds as `limbs` u32 shared atomics each at the
    measured ATOMS rate x 148 SMs x the max SM clock; (2) when `gather_stride` is given,
    one 4-byte L2 gather per add at the measured rate for lanes `gather_stride` words apart
    (the class-list gather pattern). frac = the binding ceiling's time / the kernel time."""
    if not kernel_ms:
        return None
    rows, src = _microbench_rows()
    if not rows:
        return None
    try:
        hdr = rows[0]
        best = max(r.get("ops_per_clk_per_sm", 0) for r in rows
                   if r.get("test") in ("smem_u32_atomsadd", "smem_u32_atoms_banks", "smem_u32_atoms_regs"))
        ceil = best * hdr["sms"] * hdr["clock_khz"] * 1e3
    except Exception:
        return None
    t_atom = limbs * adds / ceil
    out = {"bound": "smem_atomics", "achieved": limbs * adds / (kernel_ms * 1e-3), "peak": ceil,
           "unit": "u32 atomics/s", "limbs": limbs, "t_atomics_ms": t_atom * 1e3, "peak_source": src}
    t_bind = t_atom
    if gather_stride is not None:
        g = [r for r in rows if r.get("test") == "l2_gather_f32" and r.get("lane_stride") == gather_stride]
        if g:
            rate = g[0]["Gloads"] * 1e9
            t_g = adds / rate
            out["t_gather_ms"] = t_g * 1e3
            out["gather_loads_per_s_peak"] = rate
            out["gather_lane_stride"] = gather_stride
            if t_g > t_atom:
                out["bound"] = "l2_gather"
                t_bind = t_g
    out["frac"] = t_bind / (kernel_ms * 1e-3)
    return out


def _fp64_peaks():
    """Measured DFMA rate and 16-byte shared-memory bandwidth (microbench/fp64_peak.cu on one
    B200; the committed copy under profiles/)."""
    peak, smem = None, None
    try:
        for line in (ROOT / "profiles" / "r02_fp64_peak.jsonl").read_text().splitlines():
            d = json.loads(line)
            if d.get("test") == "dfma_peak":
                peak = max(peak or 0.0, d["tflops"])
            if d.get("test") == "smem_lds128":
                smem = max(smem or 0.0, d["TBps"])
    except (OSError, ValueError, KeyError):
        pass
    return peak, smem


def contraction_roofline(per_s, n, b, B):
    """SURVEY 8(d) model of one median-of-B T(I,u,u): 4B length-b transforms at 5 b log2 b
    nominal flops each plus B(5n + 40b). Peak: the DFMA rate measured on a B200
    (profiles/r02_fp64_peak.jsonl), else the vendor figure."""
    if not per_s:
        return None
    logb = b.bit_length() - 1
    flops = 4 * B * 5 * b * logb + B * (5 * n + 40 * b)
    tflops = per_s * flops / 1e12
    peak, smem = _fp64_peaks()
    src = "measured DFMA rate (profiles/r02_fp64_peak.jsonl)" if peak else "vendor B200 FP64 figure"
    peak = peak or 37.0
    return {"bound": "fp64", "nominal_flops_per_contraction": flops, "achieved_tflops": tflops,
            "peak_tflops": peak, "peak_source": src, "frac": tflops / peak,
            "smem_peak_tbs": smem or 148 * 128 * 1.965e9 / 1e12}


# ---------------------------------------------------------------- CPU (oracle) legs
def _oracle():
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_py as O  # CPU restatement (test/bench infrastructure), never the product

    return O


def cpu_sample_tensor(rows=REF_ROWS):
    """Rows [0, rows) of the config-2 tensor from the oracle's own generator (fp32)."""
    O = _oracle()
    c = CFG
    T, _, _ = O.gen_planted_slice(c["n"], c["rank"], c["sigma"], c["seed"], 0, rows, dtype=np.float32)
    return T


def oracle_slice_seconds(Tslice, reps, threads=None):
    """Oracle sym build (sketch.cpp:315-345) of the slice rows [0, rows) per rep."""
    O = _oracle()
    O.lib().orc_set_num_threads(threads or os.cpu_count() or 1)
    c = CFG
    rows = Tslice.shape[0]
    s = O.SymSet(c["n"], c["b"], c["B"], c["seed"])
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        s.accumulate_dense_slice(Tslice, 0, rows)
        times.append(time.perf_counter() - t0)
    # OpenMP over the B replicates: at most B threads do work (sketch.cpp:325)
    return times, min(O.lib().orc_num_threads(), c["B"])


def sample_desc(rows, threads):
    frac = simplex_entries(CFG["n"], 0, rows) / simplex_entries(CFG["n"])
    return (f"config-2 rows i in [0,{rows}) = {100 * frac:.1f}% of the sorted triples (n=1000 fp32 widened to fp64, "
            f"b=2^16, B=10) per step, oracle restatement of sketch.cpp:315-345 on {threads} threads "
            "(OpenMP over replicates); value = n^3 x sample fraction / time"), frac


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    T = cpu_sample_tensor()
    warm, _ = oracle_slice_seconds(T, max(args.warmup, 0))
    times, threads = oracle_slice_seconds(T, args.steps)
    assert not any(PRODUCT_LIB in l for l in open("/proc/self/maps")), "reference arm loaded the product library"
    desc, frac = sample_desc(T.shape[0], threads)
    tot = sum(times)
    val = CFG["n"] ** 3 * frac * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "entries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.gpus),
        "cpu_baseline": {"value": val, "unit": "entries/s", "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": val, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def config_dict(world):
    return {"workload": "config2: dense symmetric n=1000 fp32 tensor (1e9 entries, rank-100 planted, sigma=0.01), "
                        "sym sketch b=2^16 B=10",
            "n": CFG["n"], "rank": CFG["rank"], "sigma": CFG["sigma"], "b": CFG["b"], "B": CFG["B"],
            "seed": CFG["seed"], "input_dtype": "f32",
            "l2": "input (4 GB tensor, 669 MB of sorted triples) larger than L2; L2 also flushed "
                  "(256 MiB write) before every timed step",
            "parallelism": f"i-slices x{world}, exact int64 accumulators all-reduced in-library over NCCL"
            if world > 1 else "single GPU"}


# ---------------------------------------------------------------- product arm
def run_b200(args):
    import torch

    import paper_1506_04448_b200 as skb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, b, B = CFG["n"], CFG["b"], CFG["B"]
    ctx = skb.Context(local)
    ext = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    T_dev = torch.empty(n ** 3, dtype=torch.float32, device=dev)
    skb.gen_planted_tensor_device(ctx, n, CFG["rank"], CFG["sigma"], CFG["seed"], T_dev.data_ptr(), dtype=np.float32)
    i0, i1 = equal_work_slices(n, world)[rank]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sset = skb.SymTensorSketchSet(n, b, B, CFG["seed"], ctx)
    reps = None
    if world > 1 or args.group:
        # in-library NCCL (include/sketchcp_b200.h multi-GPU section): each rank builds its
        # equal-work i-slice and the exact int64 accumulators are all-reduced inside the call
        uid = [skb.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])
        reps = skb.SymReplicas(n, b, B, CFG["seed"], [ctx])
        sset = reps.sets[0]
    out_host = torch.empty((B, b), dtype=torch.complex128).pin_memory().numpy()

    def step(T, host=False):
        if reps is not None:
            reps.accumulate_dense(T if host else [T], assume_symmetric=True)
        else:
            sset.accumulate_dense(T, assume_symmetric=True)
        if host:
            return sset.data(out=out_host)
        return None

    warm = max(args.warmup, 3)
    for _ in range(warm):
        step(T_dev)
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = skb.kernel_launch_count()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            ev[k][0].record(ext)
            step(T_dev)
            ev[k][1].record(ext)
        torch.cuda.synchronize()
    launches = skb.kernel_launch_count() - launches0
    if dist:
        dist.barrier()
    ms = sum(a.elapsed_time(e) for a, e in ev)
    # per-kernel durations (roofline) from a second, identically flushed pass with the
    # library's CUDA-event scopes around each launch (they break back-to-back issue, so
    # the timed steps above run without them)
    ctx.profile(True)
    ctx.profile_reset()
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        step(T_dev)
    torch.cuda.synchronize()
    main_ms, main_cnt = ctx.profile_get("build_main")
    pre_ms, _ = ctx.profile_get("build_prepass")
    fin_ms, _ = ctx.profile_get("build_finalize")
    ctx.profile(False)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n ** 3 / (ms_step * 1e-3)
    simplex_job = simplex_entries(n)
    simplex_rank = simplex_entries(n, i0, i1)

    # ---- end-to-end through the public API: pinned host tensor in, sketch out ----------
    T_pinned = torch.empty(n ** 3, dtype=torch.float32).pin_memory()
    T_pinned.copy_(T_dev)
    T_np_pinned = T_pinned.numpy()
    for _ in range(2):  # warm the pinned (chunked pipeline) path
        step(T_np_pinned, host=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_list = []
    for k in range(max(1, min(args.steps, 10))):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        step(T_np_pinned, host=True)
        e.record(ext)
        torch.cuda.synchronize()
        e2e_list.append(a.elapsed_time(e))
    pcie = pcie_link(local)  # right after the bus-bound loop (idle links downshift)
    e2e_ms = sum(e2e_list) / len(e2e_list)
    e2e_med = statistics.median(e2e_list)
    if dist:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    del T_pinned, T_np_pinned

    # ---- config 1 (n=400 fp64): build and sketched contractions --------------------------
    c1 = extra_config1(skb, ctx, ext, flush, dev) if rank == 0 else {}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    kern_ms = main_ms / main_cnt if main_cnt else None
    achieved = simplex_rank * 4 / (kern_ms * 1e-3) / 1e9 if kern_ms else None
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded device generator, BASELINE config 2 shape)",
        "config": config_dict(world),
        "hbm_gbs_algorithmic": simplex_job * 4 / (ms_step * 1e-3) / 1e9,
        "e2e": {"value": n ** 3 / (e2e_ms * 1e-3), "unit": "entries/s",
                # pinned input: the pre-pass reads the sorted-triple rows in place over the bus
                "h2d_bytes_per_step": int(simplex_rank * 4), "d2h_bytes_per_step": int(B * b * 16),
                "ms_per_step": e2e_ms, "ms_per_step_median": e2e_med, "pcie": pcie,
                "path": "accumulate_dense(pinned host fp32 tensor) + replicate data readback into pinned host "
                        "memory (public API)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_build_cls",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic_from_profiles("k_build_cls", "config2"),
                     "algorithmic_bytes_per_launch": simplex_rank * 4,
                     "kernel_ms_per_launch": kern_ms,
                     "prepass_ms_per_launch": pre_ms / main_cnt if main_cnt else None,
                     "finalize_ms_per_launch": fin_ms / main_cnt if main_cnt else None,
                     "scatter_adds_per_s": simplex_rank * B / (kern_ms * 1e-3) if kern_ms else None,
                     "frac_vs_8tbs": (achieved / 8000.0) if achieved else None,
                     "peak_source": peak_src},
        # the ceilings the scatter actually meets (one-limb fp32 adds; gathers 4 words apart:
        # each window takes 1 of 4 (parity, bucket-parity) classes of a row's k)
        "scatter_roofline": scatter_roofline(simplex_rank * B, kern_ms, limbs=1, gather_stride=4),
        "clocks": clocks,
    }
    line.update(c1)
    if world == 1 and not args.no_cpu_baseline:
        Ts = T_dev[: REF_ROWS * n * n].cpu().numpy().reshape(REF_ROWS, n, n)  # the same entries the GPU built
        times, threads = oracle_slice_seconds(Ts, 2)
        desc, frac = sample_desc(REF_ROWS, threads)
        line["cpu_baseline"] = {"value": n ** 3 * frac / min(times), "unit": "entries/s", "cores": threads,
                                "kind": "port", "sample": desc + ", best of 2"}
        t1, _ = oracle_slice_seconds(Ts[:8], 1, threads=1)  # the paper's single-thread protocol
        line["cpu_baseline"]["single_thread_value"] = n ** 3 * simplex_entries(n, 0, 8) / simplex_entries(n) / t1[0]
        line["cpu_baseline"]["single_thread_sample"] = "rows i in [0,8) on 1 thread"
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def extra_config1(skb, ctx, ext, flush, dev):
    """Config 1 (n=400 fp64 rank 50, b=2^14, B=20): device-resident build time and the
    batched sketched contractions on its sketch (L=100 restarts)."""
    import torch

    c = CFG1
    n, b, B, L = c["n"], c["b"], c["B"], c["L"]
    T1 = torch.empty(n ** 3, dtype=torch.float64, device=dev)
    skb.gen_planted_tensor_device(ctx, n, c["rank"], c["sigma"], c["seed"], T1.data_ptr(), dtype=np.float64)
    s1 = skb.SymTensorSketchSet(n, b, B, c["seed"], ctx)
    for _ in range(3):
        s1.accumulate_dense(T1, assume_symmetric=True)
    torch.cuda.synchronize()
    steps = 10
    tms = []
    for k in range(steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        s1.accumulate_dense(T1, assume_symmetric=True)
        e.record(ext)
        torch.cuda.synchronize()
        tms.append(a.elapsed_time(e))
    ctx.profile(True)
    ctx.profile_reset()
    for k in range(steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        s1.accumulate_dense(T1, assume_symmetric=True)
    torch.cuda.synchronize()
    m_ms, m_cnt = ctx.profile_get("build_main")
    ctx.profile(False)
    build_ms = sum(tms) / len(tms)
    simplex = simplex_entries(n)
    kern = m_ms / m_cnt if m_cnt else None
    out = {"config1_build": {"workload": "config1: n=400 fp64 rank 50, sym b=2^14 B=20, device-resident, L2 flushed",
                             "entries_per_s": n ** 3 / (build_ms * 1e-3), "ms_per_step": build_ms,
                             "k_build_cls_ms": kern,
                             "hbm_frac": simplex * 8 / (kern * 1e-3) / 1e9 / peaks()[0] if kern else None,
                             "scatter_roofline": scatter_roofline(simplex * B, kern, limbs=2, gather_stride=4)}}
    # sketched contractions: batched T(I,u,u) power step (wall-clock Ivv calls on the stream)
    ws = skb.SymContractionWorkspace(s1)
    U = skb.power_inits(1, n, 1, L)[0]
    for _ in range(3):
        ws.Ivv(U)
    torch.cuda.synchronize()
    reps = 10
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ext)
    for _ in range(reps):
        ws.Ivv(U)
    e.record(ext)
    torch.cuda.synchronize()
    ivv_ms = a.elapsed_time(e) / reps
    for _ in range(2):
        ws.vvv(U)
    a.record(ext)
    for _ in range(reps):
        ws.vvv(U)
    e.record(ext)
    torch.cuda.synchronize()
    vvv_ms = a.elapsed_time(e) / reps
    per_s = L / (ivv_ms * 1e-3)
    out.update({"contractions_per_s": per_s, "contraction_step_ms": ivv_ms,
                "contraction_config": "config1 sketch, batched T(I,u,u) over L=100 restarts per Ivv call "
                                      "(host API call incl. inputs in and the n x L result out)",
                "vvv_per_s": L / (vvv_ms * 1e-3),
                "contraction_roofline": contraction_roofline(per_s, n, b, B)})
    del T1
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--group", action="store_true", help="take the multi-GPU (NCCL group) build path even at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
