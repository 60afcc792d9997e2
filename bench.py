#!/usr/bin/env python
"""bench.py — Aggregate Risk Analysis hot path on B200 (arxiv 1606.04473).

One step = one pass of the whole hot path over the
workload: ELT densify (+ NVLink broadcast when N > 1), YET ingest, the ARA
trial kernel, the YLT all-gather (N > 1) and device PML/TVaR.

  value : trials/s of the whole job with inputs already resident in HBM
          (sparse ELT lists + YET CSR on the device; the library borrows them)
  e2e   : the same step through the C-ABI with HOST buffers — pinned sparse
          ELTs + YET streamed in chunks (copy/compute overlap) and the YLT +
          metrics read back — H2D/D2H inside the timed region

N > 1: one process per GPU (torchrun); trials are sharded by ara_partition
(strong scaling of the paper-shaped layer, BASELINE config 3), the YLT is
all-gathered over NVLink.  Timing: CUDA events on the launching stream, barrier
+ synchronize on both sides, max over ranks.

--impl reference: the CPU oracle (this tier's reference arm), timed on host
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ["NCCL_DEBUG"] = os.environ.get("ARA_NCCL_DEBUG", "WARN")   # stdout: the one JSON line only

import synth  # noqa: E402

METRIC = "trials/sec and ELT lookups/sec at 1/2/4/8 B200; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="paper")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--e2e-mode", default="chunked", choices=["chunked", "all"])
    ap.add_argument("--chunk-trials", type=int, default=65536)
    ap.add_argument("--e2e-format", default="both", choices=["both", "u32"],
                    help="e2e legs: u32 host ids (the headline, plain ara_load_yet) and, with 'both', also the "
                         "bit-packed transfer format (F3, ara_load_yet_packed) as e2e_packed")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--l2-persist", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every GPU runs its own paper-shaped YET shard (N x 1M trials in all, one "
                         "global YLT, metrics over all of it); strong: the 1M trials split over the GPUs")
    ap.add_argument("--mode", default="direct", choices=["direct", "fold"],
                    help="direct = Alg. 3 per occurrence (headline); fold = catalogue-fold mode (SURVEY 8f F2)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def bind_to_gpu_numa(local: int) -> int:
    """Pin this rank to the CPUs nearest its GPU (NVML's ideal affinity), so the
    pinned host buffers allocated afterwards are first-touched on the GPU's NUMA
    node -- the host side of the paper's transfer bottleneck.  Returns
    the number of CPUs the process may run on afterwards."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        pr = torch.cuda.get_device_properties(local)
        bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        pynvml.nvmlDeviceSetCpuAffinity(h)
    except Exception:
        pass
    try:
        return len(os.sched_getaffinity(0))
    except OSError:
        return os.cpu_count() or 1


def host_info():
    cpu = "?"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": cpu, "python": platform.python_version()}


class ClockSampler:
    """SM clocks + throttle reasons (NVML every 10 ms, else nvidia-smi every
    100 ms), sampled from before the warm-up to after the timed region; mark() brackets the timed window and
    stop() summarises the samples inside it (all samples if the window was
    shorter than two sampling periods)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None
        self.win = [None, None]

    def start(self):
        # NVML polled every 10 ms (a timed region of ~10 steps lasts only
        # ~60 ms); nvidia-smi at its 100-ms floor when NVML is unavailable
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self._stop_evt = threading.Event()

            def poll():
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                while not self._stop_evt.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        act = ["Active" if r & b else "Not Active" for b in bits.values()]
                        self.lines.append((time.time(), ",".join(["t", str(self.gpu), str(sm), str(mx), "0", hex(r)] + act)))
                    except pynvml.NVMLError:
                        pass
                    time.sleep(0.01)

            self.proc = "nvml"
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.time(), ln.strip()))

    def mark(self, i):
        self.win[i] = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if self.proc == "nvml":
            time.sleep(0.03)
            self._stop_evt.set()
            self.t.join(timeout=2)
        else:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 10:
                continue
            try:
                rows.append((ts, float(p[2]), float(p[3]), [nm for nm, v in zip(names, p[6:10]) if v.lower() == "active"]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        a, b = self.win
        slack = 0.015 if self.proc == "nvml" else 0.15
        inside = [r for r in rows if a is not None and b is not None and a - slack <= r[0] <= b + slack]
        sel = inside if len(inside) >= 2 else rows
        sm = [r[1] for r in sel]
        load = [x for x in sm if x > 0.5 * max(sm)] or sm
        reasons = sorted({x for r in sel for x in r[3]})
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": float(max(r[2] for r in sel)), "reasons": reasons,
                "samples": len(sel), "window": "timed region" if sel is inside else "whole run"}


def algorithmic_bytes(w, n_events: int, n_trials: int, precision: str, mode: str = "direct",
                      occupancy: float = 1.0, packed: bool = False) -> dict:
    """DESIGN.md section 6 "Algorithmic bytes", the north star's count: YET
    bytes streamed + 32 B per ELT sector the kernel actually gathers, per
    launch (layers sharing one row window share a launch).  Direct mode: per
    event 4 B of id; per gathered event the row window's 32-B sectors -- or,
    with packed rows (the sparse kernel), one 32-B slot for the occupied
    fraction of events only (an unoccupied row is never read); per trial 8 B
    of offsets + 8 B per YLT row.  The occupancy probes (one bit per event,
    a 250 KB bitmap held in shared memory / L1 / L2, never DRAM-streamed) are
    NOT HBM bytes: they are returned separately as index_bytes (one 4-B word
    per probe).  Fold mode: the fold pass reads every catalogue row window
    once and writes 8 B per (event id, layer); the trial pass reads 4 B of id
    + one fold row (8 B x layers, padded to a power of two) per event -- per
    occupied event for the sparse fold pass (variant 31)."""
    eps = 4 if precision == "f64" else 8
    windows = []
    for L in w.layers:
        win = (L.elt_begin // eps, (L.elt_end + eps - 1) // eps)
        if not windows or windows[-1][0] != win or windows[-1][1] == 4:
            windows.append([win, 1])
        else:
            windows[-1][1] += 1
    per_trial = n_trials * (8 + 8 * (len(w.layers) + 1))
    if mode == "fold":
        sec = sum(b - a for (a, b), _ in windows)
        nl = len(w.layers)
        nlc = 1
        while nlc < nl and nlc < 8:
            nlc *= 2
        # the sparse fold pass (variant 31) gathers the fold row of the occupied
        # events only; the dense one gathers it for every event
        frac = occupancy if packed else 1.0
        hbm = int((w.catalog + 1) * (32 * sec + 8 * nl) + n_events * (4 + frac * 8 * nlc) * ((nl + nlc - 1) // nlc)
                  + per_trial)
        return {"hbm": hbm, "index": 0, "yet": 4 * n_events * ((nl + nlc - 1) // nlc), "elt": hbm - per_trial}
    yet = elt = index = 0.0
    for (a, b), _ in windows:
        yet += 4.0 * n_events
        if packed:
            elt += occupancy * 32.0 * n_events
            index += 4.0 * n_events
        else:
            elt += 32.0 * (b - a) * n_events
    return {"hbm": int(yet + elt + per_trial), "index": int(index), "yet": int(yet), "elt": int(elt),
            "per_trial": int(per_trial)}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


KERNEL_NAMES = {30: "ara::trial_kernel_bc (ballot-compacted rounds over packed rows)",
                12: "ara::trial_kernel_co (cooperative ring)",
                5: "ara::trial_kernel (register pipeline)", 0: "ara::trial_kernel (register pipeline)",
                -2: "ara::fold_kernel+trial_fold_kernel",
                31: "ara::fold_kernel+trial_kernel_bc<fold> (rounds gather o(e) of the occupied events)"}


def kernel_name(variant):
    """The trial kernel the library reports it launched (ara_run_stats.kernel_variant)."""
    return KERNEL_NAMES.get(int(variant), f"ara::trial_kernel (ARA_KERNEL={variant})")


L2_PEAK_SOURCE = "profiles/r01_microbench.json"


def l2_gather_peak():
    """Builder-measured L2 gather ceiling (GB/s): random 32-B gathers from an
    L2-resident 16 MB table (tools/microbench.py); not a MEASURED_PEAKS.json
    figure, so every use names the file."""
    try:
        return json.load(open(os.path.join(ROOT, L2_PEAK_SOURCE)))["gather_16MB_32B_gbs"]
    except (OSError, ValueError, KeyError):
        return None


def issue_roofline(trec, k_ms, clk, dev):
    """Instruction-issue roofline of the dominant kernel: warp instructions per
    launch (ncu, profiles/ara_kernel_traffic.json, same kernel and launch size)
    over the kernel time, against 4 warp instructions per SM per cycle (one per
    SM sub-partition) x SMs x the SM clock sampled during the timed region."""
    if not trec or not trec.get("warp_instructions_per_launch") or not clk or not clk.get("sm_mhz"):
        return None
    import torch
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    achieved = trec["warp_instructions_per_launch"] / (k_ms / 1e3)
    peak = 4.0 * n_sm * clk["sm_mhz"] * 1e6
    return {"achieved": achieved, "peak": peak, "unit": "warp instructions/s", "frac": achieved / peak,
            "instructions_per_launch": trec["warp_instructions_per_launch"], "sms": n_sm,
            "sm_mhz": clk["sm_mhz"], "source": trec.get("source")}


def load_traffic(w, precision, variant, n_trials_launch):
    """DRAM bytes and L2->SM sectors per launch of the ARA kernel from the
    committed ncu --set full capture of the same kernel variant AT THE SAME
    LAUNCH SIZE (trials per launch), or None."""
    p = os.path.join(ROOT, "profiles", "ara_kernel_traffic.json")
    try:
        d = json.load(open(p)).get(f"{w.name}/{precision}", {})
    except (OSError, ValueError):
        return None
    if d.get("variant") != variant or d.get("n_trials_per_launch") != n_trials_launch:
        return None
    return d


# ------------------------------------------------------------------ oracle (cpu baseline / reference arm)
def oracle_sample_rate(w, seconds: float, precision: str):
    """The oracle as it stands (single thread, dense direct-access lookups) on
    the first trials of the workload; sized to ~`seconds` of CPU work."""
    import oracle
    eo, ev, ls = synth.gen_elts(w)
    E = oracle.Elts(eo, ev, ls)
    dense = oracle.direct_access(E, w.catalog)
    d, li = w.elt_terms()
    lay = oracle.layers_from_specs(w.layers)

    def run(n):
        off, ids = synth.gen_yet(w, first=0, n=n)
        t0 = time.perf_counter()
        oracle.ara(off, ids, E, w.catalog, d, li, lay, lookup="dense", dense=dense,
                   fp32_storage=precision == "f32")
        return time.perf_counter() - t0, int(off[-1])

    t, _ = run(200)
    n = int(max(200, min(w.n_trials, 200 * seconds / max(t, 1e-6))))
    t, ev_n = run(n)
    return {"trials": n, "seconds": t, "trials_per_s": n / t, "events": ev_n,
            "lookups_per_s": ev_n * sum(L.elt_end - L.elt_begin for L in w.layers) / t}


def reference_arm(a, rank, world):
    if rank != 0:
        return
    w = synth.get_config(a.config)
    per_step = max(2.0, 60.0 / max(1, a.steps + a.warmup))
    res = []
    for i in range(a.warmup + a.steps):
        r = oracle_sample_rate(w, per_step, a.precision)
        if i >= a.warmup:
            res.append(r)
    tps = float(np.median([r["trials_per_s"] for r in res]))
    sample = f"first {res[0]['trials']} trials of the {w.name} workload per step, dense direct-access lookups"
    # the same config as our arm (weak scaling: N x the workload's trials); the
    # oracle's rate is measured on the bounded sample above
    n_trials = w.n_trials * (world if a.scaling == "weak" else 1)
    # ms_per_step is the MEASURED time of one step (one bounded sample); the
    # time the oracle would need for the whole workload is a projection
    line = {"impl": "reference", "metric": METRIC, "value": tps, "unit": "trials/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * float(np.median([r["seconds"] for r in res])),
            "ms_per_step_projected_full_workload": 1e3 * n_trials / tps,
            "trials_per_step": int(np.median([r["trials"] for r in res])),
            "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": a.precision,
            "data": "synthetic", "config": {"workload": w.name, "n_trials": n_trials},
            "lookups_per_sec": float(np.median([r["lookups_per_s"] for r in res])),
            "cpu_baseline": {"value": tps, "unit": "trials/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": tps, "unit": "trials/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "host": host_info()}
    emit(line)


# ------------------------------------------------------------------ our arm
_JSON_FD = None


def emit(line: dict):
    """The one stdout line of the bench contract.  Library/NCCL chatter written
    to fd 1 by C code is routed to stderr (see main), so this write is the only
    thing on the original stdout."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is not None:
        os.write(_JSON_FD, data)
    else:
        sys.stdout.write(data.decode())
        sys.stdout.flush()


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)          # anything else printed to fd 1 (NCCL version banners, ...) goes to stderr
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return reference_arm(a, rank, world)

    import torch
    import torch.distributed as dist
    from paper_1606_04473_b200 import ara

    torch.cuda.set_device(local)
    cpus_bound = bind_to_gpu_numa(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = synth.get_config(a.config)
    trials_per_gpu = w.n_trials
    if a.scaling == "weak":   # N x the workload's trials; rank r holds trials [r T1, (r+1) T1)
        w = w.with_(n_trials=w.n_trials * world)
    else:
        trials_per_gpu = (w.n_trials + world - 1) // world
    T = w.n_trials
    first, count = ara.ara_partition(T, world, rank)
    stream = torch.cuda.current_stream()

    def new_nccl_id():
        """A fresh NCCL unique id per communicator (an id initialises one communicator)."""
        if world == 1:
            return None
        obj = [ara.ara_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs: this rank's YET shard generated straight into pinned memory
    t_gen = time.time()
    n_off = count + 1
    off_pin = torch.empty(n_off, dtype=torch.int64, pin_memory=True)
    synth.gen_offsets(w, first, count, out=off_pin.numpy().view(np.uint64))
    n_ev = int(off_pin[-1])
    ids_pin = torch.empty(max(n_ev, 1), dtype=torch.int32, pin_memory=True)
    synth.gen_events(w, synth.event_base(w, first), n_ev, out=ids_pin.numpy().view(np.uint32))
    if rank == 0:
        eo, ev, ls = synth.gen_elts(w)
        eo_pin = torch.from_numpy(eo.view(np.int64)).pin_memory()
        ev_pin = torch.from_numpy(ev.view(np.int32)).pin_memory()
        ls_pin = torch.from_numpy(ls).pin_memory()
        d_eo, d_ev, d_ls = eo_pin.to(dev), ev_pin.to(dev), ls_pin.to(dev)
    else:
        eo_pin = ev_pin = ls_pin = d_eo = d_ev = d_ls = None
    d_off = off_pin.to(dev)
    d_ids = ids_pin[:n_ev].to(dev) if n_ev else ids_pin.to(dev)
    torch.cuda.synchronize()
    gen_s = time.time() - t_gen
    terms = w.elt_terms()
    R = list(w.return_periods)
    L = len(w.layers)

    # ---- device-resident arm (value)
    ctx = ara.Context(w.catalog, device=local, precision=a.precision, stream=stream, rank=rank, world=world,
                      nccl_id=new_nccl_id(), l2_persist=a.l2_persist, run_mode=a.mode)
    kern_ms, ag_ms, met_ms, launches = [], [], [], []
    used = {}

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    part_ms = []

    def step(record):
        evs[0].record(stream)
        ctx.load_elts(d_eo, d_ev, d_ls, terms, n_elts=w.n_elts)          # a0 (+ NVLink broadcast)
        evs[1].record(stream)
        ctx.load_yet(T, first, d_off, d_ids)                             # a1 (device: borrowed)
        evs[2].record(stream)
        st = ctx.run(w.layers)                                           # a2-a9
        evs[3].record(stream)
        k, pml, tvar, mms = ctx.metrics(R)                               # a10
        evs[4].record(stream)
        if record:
            kern_ms.append(st["kernel_ms"])
            ag_ms.append(st["allgather_ms"])
            met_ms.append(mms)
            launches.append(st["n_kernel_launches"])
            used.update(variant=st["kernel_variant"], occupancy=st["occupancy"])
            evs[4].synchronize()
            part_ms.append([evs[i].elapsed_time(evs[i + 1]) for i in range(4)])
        return st, pml, tvar

    clocks = ClockSampler(local)
    clocks.start()                       # sampling runs from warm-up through the timed region
    for _ in range(a.warmup):
        st0, pml, tvar = step(False)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark(0)
    e0.record(stream)
    for _ in range(a.steps):
        st, pml, tvar = step(True)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(1)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1)) / a.steps
    ev_local = st["n_events_local"]
    if world > 1:
        t = torch.tensor([ev_local], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        n_events_global = int(t.item())
    else:
        n_events_global = ev_local
    lookups = n_events_global * sum(Lr.elt_end - Lr.elt_begin for Lr in w.layers)
    value = T / (ms / 1e3)

    # roofline of the dominant kernel (the ARA trial kernel) on this rank
    k_ms = float(np.mean(kern_ms))
    algb = algorithmic_bytes(w, ev_local, count, a.precision, a.mode, occupancy=used.get("occupancy", 1.0),
                             packed=used.get("variant") in (30, 31))
    alg = algb["hbm"]
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)"
    if not peak:
        peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    achieved = alg / (k_ms / 1e3) / 1e9
    trec = load_traffic(w, a.precision, used.get("variant"), count) if a.mode == "direct" else None
    traffic = trec.get("dram_bytes_per_launch") if trec else None
    l2pk = l2_gather_peak()
    ctx.close()

    # ---- end-to-end arm: host buffers through the C-ABI
    e2e = None
    def e2e_leg(fmt):
        """The step through the C-ABI with pinned HOST buffers: ELT records + YET
        (u32 ids, or the F3 packed transfer format) copied in chunks overlapped
        with the kernel, YLT + metrics read back, all inside the timed region."""
        ylt_pin = torch.empty((L + 1) * T, dtype=torch.float64, pin_memory=True)
        ids_view = ids_pin[:n_ev]
        bits = ara.bits_for_catalog(w.catalog)
        pack_ms = None
        if fmt == "packed":   # host YET stored in the packed transfer format (setup, untimed; timed once below)
            packed_pin = torch.empty(ara.ara_packed_words(n_ev, bits), dtype=torch.int32, pin_memory=True)
            tp = time.perf_counter()
            ara.ara_pack_ids(ids_pin.numpy().view(np.uint32)[:n_ev], bits, packed_pin)
            pack_ms = 1e3 * (time.perf_counter() - tp)
            ids_bytes = packed_pin.numel() * 4
        else:
            ids_bytes = n_ev * 4
        ectx = ara.Context(w.catalog, device=local, precision=a.precision, stream=stream, rank=rank, world=world,
                           nccl_id=new_nccl_id(), load_mode=a.e2e_mode, chunk_trials=a.chunk_trials,
                           l2_persist=a.l2_persist, run_mode=a.mode)
        h2d_ms = []
        wall = []

        def estep():
            t0 = time.perf_counter()
            ectx.load_elts(eo_pin, ev_pin, ls_pin, terms, n_elts=w.n_elts)
            t1 = time.perf_counter()
            if fmt == "packed":
                ectx.load_yet_packed(T, first, off_pin, packed_pin, bits)
            else:
                ectx.load_yet(T, first, off_pin, ids_view)
            t2 = time.perf_counter()
            s2 = ectx.run(w.layers, ylt_pin)
            t3 = time.perf_counter()
            ectx.metrics(R)
            t4 = time.perf_counter()
            h2d_ms.append(s2["h2d_ms"])
            wall.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
            return s2

        for _ in range(max(1, a.warmup)):
            estep()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(a.steps):
            estep()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1)) / a.steps
        h2d = n_off * 8 + ids_bytes + (eo_pin.numel() * 8 + ev_pin.numel() * 4 + ls_pin.numel() * 8 if rank == 0 else 0)
        d2h = (L + 1) * T * 8 + 2 * (L + 1) * len(R) * 8 + 8
        ectx.close()
        return {"value": T / (ems / 1e3), "unit": "trials/s", "ms_per_step": ems, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "mode": a.e2e_mode, "chunk_trials": a.chunk_trials,
                "yet_format": fmt + (str(bits) if fmt == "packed" else ""),
                "host_pack_ms_untimed": pack_ms,
                "h2d_gbs": (ids_bytes + n_off * 8) / (float(np.mean(h2d_ms[-a.steps:])) / 1e3) / 1e9
                if a.e2e_mode == "chunked" and np.mean(h2d_ms) > 0 else None,
                "wall_ms": {k: 1e3 * float(np.median([x[i] for x in wall[-a.steps:]]))
                            for i, k in enumerate(("load_elts", "load_yet", "run", "metrics"))}}

    # ---- end-to-end arm: host buffers through the C-ABI.  The headline e2e is
    # the plain u32 contract of ara_load_yet; e2e_packed is the same step with
    # the host YET held in the 21-bit transfer format (F3)
    e2e = e2e_packed = None
    if not a.no_e2e:
        e2e = e2e_leg("u32")
        if a.e2e_format == "both":
            e2e_packed = e2e_leg("packed")

    # ---- CPU baseline (oracle) on rank 0 at N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        r = oracle_sample_rate(w, a.cpu_seconds, a.precision)
        cpu = {"value": r["trials_per_s"], "unit": "trials/s", "cores": 1, "kind": "oracle",
               "sample": f"first {r['trials']} trials ({r['events']} events) of the {w.name} workload, "
                         f"single-threaded, dense direct-access lookups, {r['seconds']:.1f} s",
               "lookups_per_s": r["lookups_per_s"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "trials/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": a.precision, "data": "synthetic",
            "config": {"workload": w.name, "n_trials": T, "trials_per_gpu": trials_per_gpu,
                       "events_per_trial": [w.nmin, w.nmax],
                       "n_events": n_events_global, "elts_per_layer": [Lr.elt_end - Lr.elt_begin for Lr in w.layers],
                       "catalog": w.catalog, "layers": L, "return_periods": len(R), "parallelism": f"trials/{world}",
                       "l2": "inputs larger than L2 (4 GB YET streamed once per step; 256 MB table)",
                       "l2_persist": a.l2_persist, "mode": a.mode, "rho": w.rho,
                       "occupied_fraction": used.get("occupancy")},
            "lookups_per_sec": lookups / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_name(used.get("variant", -1)),
                         "kernel_ms": k_ms, "algorithmic_bytes_per_launch": alg,
                         "algorithmic_bytes": {"yet": algb["yet"], "elt_sectors": algb["elt"],
                                               "offsets_ylt": algb.get("per_trial", 0)},
                         # one 4-B bitmap word per event: shared memory / L1 / L2, never HBM-streamed
                         "index_bytes": algb["index"], "peak_source": peak_src,
                         # from the committed ncu capture of the same kernel at the same launch
                         # size (profiles/ara_kernel_traffic.json), else null
                         "dram_achieved": (traffic / (k_ms * 1e6)) if traffic else None,
                         "dram_frac": (traffic / (k_ms * 1e6) / peak) if traffic else None,
                         "l2_hit_rate_pct": trec.get("l2_hit_rate_pct") if trec else None,
                         "l2_sector_bytes": (32 * trec["l2_sectors_per_launch"]) if trec else None,
                         "l2_peak_gbs": l2pk, "l2_peak_source": L2_PEAK_SOURCE + " (builder microbenchmark: "
                                                                  "random 32-B gathers, L2-resident 16 MB table)",
                         "l2_frac": (32 * trec["l2_sectors_per_launch"] / (k_ms * 1e6) / l2pk)
                         if (trec and l2pk) else None,
                         "traffic_source": trec.get("source") if trec else None,
                         # SURVEY 8(d) F_roof: the larger of the DRAM time (ncu DRAM bytes / HBM
                         # peak) and the L2 time (ncu L2 sector bytes / L2 gather ceiling), over
                         # the kernel time
                         "hierarchical_frac": (max(traffic / peak, 32 * trec["l2_sectors_per_launch"] / l2pk)
                                               / 1e6 / k_ms) if (trec and l2pk) else None,
                         "note": ("frac = north-star bytes (YET ids + the 32-B ELT sectors actually gathered "
                                  "+ offsets/YLT) / kernel time / HBM peak; occupancy probes are index_bytes, "
                                  "not HBM bytes"),
                         # the kernel's binding limit is instruction issue, not HBM: warp instructions
                         # per launch (same ncu capture) / kernel time vs one warp instruction per
                         # cycle per SM sub-partition (4 per SM) at the SM clock sampled in the run
                         "issue": issue_roofline(trec, k_ms, clk, dev)},
            "breakdown_ms": {"ara_kernel": k_ms, "allgather": float(np.mean(ag_ms)), "metrics": float(np.mean(met_ms)),
                             "step": ms,
                             "calls": {k: float(np.median([p[i] for p in part_ms]))
                                       for i, k in enumerate(("load_elts", "load_yet", "run", "metrics"))}},
            # our kernels per timed step: load_elts = clear_rows (the table was densified
            # before) + densify + pack_rows; ara_run = n_kernel_launches; ara_metrics =
            # init + 8 radix passes + tail
            "gpu_launches": int(a.steps * (3 + np.mean(launches) + 10)),
            "e2e": e2e, "e2e_packed": e2e_packed, "cpu_baseline": cpu, "clocks": clk,
            "host": dict(host_info(), cpus_near_gpu=cpus_bound), "gen_seconds": gen_s,
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
