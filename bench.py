#!/usr/bin/env python
"""Benchmark of the FFT tensor-sketch hot path (BASELINE.json metric:
"tensor-sketch build entries/s (HBM GB/s) and sketched T(I,u,u) contractions/s").

Workload (N=1 and every N): BASELINE config 1 — dense symmetric n=400 fp64 tensor,
rank-50 planted + 0.01 mirrored Gaussian noise (host generator, seeded), symmetric
sketch b=2^14, B=20. One step = one full sketch build of the tensor (sorted
triples, sketch.cpp:315-345) resident in HBM; with N ranks the i-slices are split
by equal work and the B x b sketches are summed with an NCCL all-reduce (strong
scaling). `value` = n^3 logical entries per second for the whole job. The
sketched-contraction throughput (batched T(I,u,u), L=100 restarts, the RTPM power
step) is reported beside it.

--impl reference times the reference algorithm's CPU implementation (the oracle
restatement, oracle/; the reference itself cannot be built here) on the host
cores, rank 0 only.
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
CFG = dict(n=400, rank=50, sigma=0.01, b=1 << 14, B=20, seed=20150615, L=100)


def simplex_entries(n, i0=0, i1=None):
    i1 = n if i1 is None else i1
    return sum((n - i) * (n - i + 1) // 2 for i in range(i0, i1))


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


def traffic_from_profiles(kernel):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        e = d.get(kernel)
        if e and e.get("config") == "config1":
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


def scatter_roofline(adds, kernel_ms):
    """Exact adds as 2 random u32 shared atomics each, against the measured random ATOMS
    ceiling (microbench/atomics.cu: ops/clk/SM at 4 CTAs/SM) x 148 SMs x the max SM clock."""
    if not kernel_ms:
        return None
    ceil = None
    p = ROOT / "profiles" / "r01_microbench_atomics.jsonl"
    try:
        rows = [json.loads(l) for l in p.read_text().splitlines() if l.strip()]
        hdr = rows[0]
        best = max(r["ops_per_clk_per_sm"] for r in rows if r.get("test") == "smem_u32_atomsadd")
        ceil = best * hdr["sms"] * hdr["clock_khz"] * 1e3
    except Exception:
        return None
    achieved = 2.0 * adds / (kernel_ms * 1e-3)
    return {"bound": "smem_atomics", "achieved": achieved, "peak": ceil, "unit": "u32 atomics/s",
            "frac": achieved / ceil, "peak_source": "profiles/r01_microbench_atomics.jsonl"}


def contraction_roofline(per_s, n, b, B):
    """SURVEY 8(d) model of one median-of-B T(I,u,u): 4B length-b transforms at 5 b log2 b
    nominal flops each plus B(5n + 40b); shared memory moves 32b bytes per radix-2 pass
    equivalent of each transform (radix-R: 32b ceil(log2 b / log2 R), R=2 is the upper
    model). Peaks: FP64 vendor figure (not measured here) and 148 SMs x 128 B/clk at the
    1965 MHz SM clock."""
    if not per_s:
        return None
    logb = b.bit_length() - 1
    flops = 4 * B * 5 * b * logb + B * (5 * n + 40 * b)
    tflops = per_s * flops / 1e12
    return {"bound": "fp64", "nominal_flops_per_contraction": flops, "achieved_tflops": tflops,
            "peak_tflops": 37.0, "peak_source": "vendor B200 FP64 figure", "frac": tflops / 37.0,
            "smem_peak_tbs": 148 * 128 * 1.965e9 / 1e12}


def oracle_build_seconds(T, reps, threads=None):
    """Oracle (CPU restatement) sym build of the whole tensor with all host threads (or
    `threads`)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_py as O

    O.lib().orc_set_num_threads(threads or os.cpu_count() or 1)
    times = []
    for _ in range(reps):
        s = O.SymSet(CFG["n"], CFG["b"], CFG["B"], CFG["seed"])
        t0 = time.perf_counter()
        s.accumulate_dense(T, assume_symmetric=True)
        times.append(time.perf_counter() - t0)
    return times, O.lib().orc_num_threads()


def make_tensor():
    import paper_1506_04448_b200 as skb

    T, lam, V = skb.gen_planted_tensor(CFG["n"], CFG["rank"], CFG["sigma"], CFG["seed"])
    return T


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    T = make_tensor()
    n = CFG["n"]
    warm, _ = oracle_build_seconds(T, max(args.warmup, 0))
    times, threads = oracle_build_seconds(T, args.steps)
    tot = sum(times)
    val = n ** 3 * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "entries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.gpus),
        "cpu_baseline": {"value": val, "unit": "entries/s", "cores": threads, "kind": "port",
                         "sample": "full config-1 build (n=400, b=2^14, B=20) per step, oracle restatement "
                                   "of sketch.cpp:315-345 (reference not buildable: no Eigen3/FFTW3)"},
        "e2e": {"value": val, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def config_dict(world):
    return {"workload": "config1: dense symmetric n=400 fp64 tensor (rank-50 planted, sigma=0.01), "
                        "sym sketch b=2^14 B=20; contractions: batched T(I,u,u) over L=100 restarts",
            "n": CFG["n"], "rank": CFG["rank"], "sigma": CFG["sigma"], "b": CFG["b"], "B": CFG["B"],
            "seed": CFG["seed"], "L": CFG["L"],
            "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": f"i-slices x{world} + NCCL all-reduce" if world > 1 else "single GPU"}


def run_b200(args):
    import torch

    import paper_1506_04448_b200 as skb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, b, B = CFG["n"], CFG["b"], CFG["B"]
    ctx = skb.Context(local)
    ext = torch.cuda.ExternalStream(ctx.stream())
    T_host = make_tensor()
    T_pinned = torch.from_numpy(T_host).pin_memory()
    T_dev = T_pinned.to(f"cuda:{local}")
    from paper_1506_04448_b200.distributed import equal_work_slices

    i0, i1 = equal_work_slices(n, world)[rank]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    sset = skb.SymTensorSketchSet(n, b, B, CFG["seed"], ctx)
    dptr, dbytes = sset.data_device()

    class _CAI:  # zero-copy torch view of the set's device data for the collective
        __cuda_array_interface__ = {"shape": (dbytes // 8,), "typestr": "<f8", "data": (dptr, False), "version": 3}

    data_view = torch.as_tensor(_CAI(), device=f"cuda:{local}")

    # pinned host buffer for the per-step sketch readback of the end-to-end leg
    out_host = torch.empty((B, b), dtype=torch.complex128).pin_memory().numpy()

    def step(T, host=False):
        if world > 1 and rank != 0:
            with torch.cuda.stream(ext):
                data_view.zero_()  # prior sketch counted once by the all-reduce
        sset.accumulate_dense(T, assume_symmetric=True, i0=i0, i1=i1)
        if world > 1:
            with torch.cuda.stream(ext):
                dist.all_reduce(data_view)
            sset.bump_version()
        if host:
            return sset.data(out=out_host)
        return None

    for _ in range(max(args.warmup, 3)):
        step(T_dev)
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # (the library's per-kernel profiling events stay off here: an event recorded between
    # two launches costs the step ~40 us of back-to-back launch overlap)
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
    # library's CUDA-event scopes around each launch
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
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n ** 3 / (ms_step * 1e-3)
    simplex_bytes_job = simplex_entries(n) * 8
    simplex_bytes_rank = simplex_entries(n, i0, i1) * 8

    # ---- end-to-end through the public API: pinned host tensor in, sketch out ----------
    T_np_pinned = T_pinned.numpy()
    for _ in range(max(args.warmup, 3)):  # warm the pinned (chunked pipeline) path too
        step(T_np_pinned, host=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_ev = []
    for k in range(max(1, args.steps)):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        step(T_np_pinned, host=True)
        e.record(ext)
        e2e_ev.append((a, e))
    torch.cuda.synchronize()
    pcie = pcie_link(local)  # right after the bus-bound loop (idle links downshift)
    e2e_list = [a.elapsed_time(e) for a, e in e2e_ev]
    e2e_ms = sum(e2e_list) / len(e2e_list)
    e2e_med = statistics.median(e2e_list)
    if dist:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- sketched contractions: batched T(I,u,u) power step over L restarts -----------
    L = CFG["L"]
    ws = skb.SymContractionWorkspace(sset)
    U = skb.power_inits(1, n, 1, L)[0]
    for _ in range(2):
        ws.Ivv(U)
    ctx.profile(True)
    ctx.profile_reset()
    reps = 10
    for _ in range(reps):
        ws.Ivv(U)
    c_ms, _ = ctx.profile_get("sym_contract")
    m_ms, _ = ctx.profile_get("median")
    ctx.profile(False)
    contr_per_s = L * reps / ((c_ms + m_ms) * 1e-3) if (c_ms + m_ms) > 0 else None
    # T(u,u,u) (the RTPM restart selection): 2B forward transforms per vector
    for _ in range(2):
        ws.vvv(U)
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(reps):
        ws.vvv(U)
    v_ms = ctx.profile_get("sym_contract")[0] + ctx.profile_get("vvv_finish")[0]
    ctx.profile(False)
    vvv_per_s = L * reps / (v_ms * 1e-3) if v_ms > 0 else None

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    achieved = simplex_bytes_rank / (main_ms / main_cnt * 1e-3) / 1e9 if main_cnt else None
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded host generator, BASELINE config 1 shape)",
        "config": config_dict(world),
        "hbm_gbs_algorithmic": simplex_bytes_job / (ms_step * 1e-3) / 1e9,
        "contractions_per_s": contr_per_s,
        "contraction_step_ms": (c_ms + m_ms) / reps,
        "vvv_per_s": vvv_per_s,
        "contraction_roofline": contraction_roofline(contr_per_s, n, b, B),
        "e2e": {"value": n ** 3 / (e2e_ms * 1e-3), "unit": "entries/s",
                # pinned input: the quantize pass reads the sorted-triple rows in place over the bus
                "h2d_bytes_per_step": int(simplex_bytes_job), "d2h_bytes_per_step": int(B * b * 16),
                "ms_per_step": e2e_ms, "ms_per_step_median": e2e_med, "pcie": pcie,
                "path": "accumulate_dense(pinned host tensor) + replicate data readback into pinned host memory (public API)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_build_cls",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic_from_profiles("k_build_cls"),
                     "algorithmic_bytes_per_launch": simplex_bytes_rank,
                     "kernel_ms_per_launch": main_ms / main_cnt if main_cnt else None,
                     "prepass_ms_per_launch": pre_ms / main_cnt if main_cnt else None,
                     "finalize_ms_per_launch": fin_ms / main_cnt if main_cnt else None,
                     "scatter_adds_per_s": (simplex_entries(n, i0, i1) * B) / (main_ms / main_cnt * 1e-3) if main_cnt else None,
                     "frac_vs_8tbs": (achieved / 8000.0) if achieved else None,
                     "peak_source": peak_src},
        # the ceiling the scatter actually meets: random u32 shared-memory atomics (two
        # exact limbs per add), against the microbenchmarked rate (profiles/r01_microbench_atomics.jsonl)
        "scatter_roofline": scatter_roofline(simplex_entries(n, i0, i1) * B, main_ms / main_cnt if main_cnt else None),
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        times, threads = oracle_build_seconds(T_host, 2)
        best = min(times)
        line["cpu_baseline"] = {"value": n ** 3 / best, "unit": "entries/s", "cores": threads, "kind": "port",
                                "sample": "full config-1 build (n=400, b=2^14, B=20), best of 2, oracle restatement"}
        # the paper's single-thread protocol: one full build on one core
        t1, _ = oracle_build_seconds(T_host, 1, threads=1)
        line["cpu_baseline"]["single_thread_value"] = n ** 3 / t1[0]
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
