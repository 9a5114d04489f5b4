#!/usr/bin/env python3
"""Benchmark of the Squares RNG hot path on B200 (BASELINE.json metric:
"Gsamples/s per GPU and box (1/2/4/8 B200); % HBM write BW or % IMAD peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4|c5] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step is one pass of the hot path over one batch: for the default workload c2
(BASELINE.json configs[1]: squares32, one key from seed 1, counters 0..2^30-1, uint32 output,
4 GiB) one sq_fill_u32 launch over this rank's contiguous counter shard.  `value` is the
whole-job throughput (samples of all ranks / max-over-ranks device time), inputs resident.
`e2e` is the same metric through the C ABI with HOST buffers (sq_fill_host: chunked generation
+ D2H into pinned memory, copies inside the timed region).  `--impl reference` times the CPU
oracle (the tier's reference arm) on the host cores.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth_inputs as SI  # noqa: E402

METRIC = "Gsamples/s per GPU and box (1/2/4/8 B200); % HBM write BW or % IMAD peak"
UNIT = "Gsamples/s"
FALLBACK_HBM_GBS = 6650.0          # /opt/skills/guides/B200_PROFILING.md fallback
SM_PER_GPU = 148


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0}, "fallback"


def load_profile_summary():
    """Per-kernel ncu figures committed under profiles/ (traffic = dram read+write per launch)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampler of SM clock and clock-event (throttle) reasons DURING the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x40: "sw_thermal_slowdown",
               0x80: "hw_thermal_slowdown", 0x100: "hw_power_brake_slowdown", 0x2: "applications_clocks",
               0x20: "sync_boost", 0x1: "gpu_idle"}

    def __init__(self, torch_dev: int, interval_s: float = 0.005):
        self.samples, self.reasons, self.ok, self.power = [], set(), False, []
        self.interval = interval_s
        self._stop = threading.Event()
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(torch_dev)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                except Exception:
                    pass
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.interval)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "")}
        out = {"sm_mhz": statistics.median(self.samples) if self.samples else None,
               "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power:
            out["power_w_median"] = statistics.median(self.power)
            out["power_w_max"] = max(self.power)
        return out


# ------------------------------------------------------------------------------------- CPU oracle
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    """The host CPU's model name (lscpu's "Model name"; /proc/cpuinfo on Linux)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_keys(w: SI.Workload, count: int):
    """The workload's keys from the ORACLE's key utility (the reference arm and cpu_baseline
    never load the product; tests/test_capi_host.py checks both key utilities agree)."""
    import oracle as O
    return [int(k) for k in O.keygen(w.key_seed, count)]


def oracle_rate(w: SI.Workload, key: int, keys, budget_s: float, threads: int):
    """Times the oracle AS IT STANDS (oracle/oracle.c, gcc -O2, one loop per thread) on a
    bounded sample of workload w: `threads` disjoint contiguous shards of its counter range
    (or key rows), each about `budget_s` seconds of one core.  Output buffers are allocated and
    first touched, and the thread pool started, BEFORE the timed window (no page faults or
    thread start-up inside it).  Returns (samples/s, samples, wall seconds, description)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle as O
    kind = w.kind
    # calibrate on one thread
    m0 = 1 << 18
    t0 = time.perf_counter()
    if kind == "fused":
        O.fused_stats(key, 0, m0)
    else:
        O.fill(kind, [key], 0, m0)
    r1 = m0 / max(time.perf_counter() - t0, 1e-6)
    per = int(max(1 << 16, min(r1 * budget_s, w.samples // threads)))
    M64 = (1 << 64) - 1
    lib = O.lib()
    if w.nkeys > 1:
        # multi-key workload: each thread fills whole rows (one key each, n counters per row)
        rows = max(1, per // w.n)
        per = rows * w.n
        kk = [np.array([int(keys[(i * rows + r) % len(keys)]) & M64 for r in range(rows)], dtype=np.uint64)
              for i in range(threads)]
    else:
        kk = [np.array([key & M64], dtype=np.uint64) for _ in range(threads)]
        rows = 1
    bufs = [None] * threads
    hs = [np.zeros(65536, np.uint64) for _ in range(threads)] if kind == "fused" else None
    os_ = [np.zeros(32, np.uint64) for _ in range(threads)] if kind == "fused" else None
    if kind != "fused":
        dt = {"u32": np.uint32, "u64": np.uint64, "f32": np.float32}[kind]
        bufs = [np.empty(per, dtype=dt) for _ in range(threads)]
        for b in bufs:
            b.fill(0)   # write every page now (np.zeros may map lazily-zeroed pages)
    fn = None if kind == "fused" else getattr(lib, f"oracle_fill_{kind}")

    def work(i):
        if kind == "fused":
            lib.oracle_fused_stats(key & M64, (w.samples // threads) * i, per, hs[i].ctypes.data, os_[i].ctypes.data)
        elif w.nkeys > 1:
            fn(kk[i].ctypes.data, rows, w.ctr0, w.n, bufs[i].ctypes.data, w.n)
        else:
            fn(kk[i].ctypes.data, 1, (w.samples // threads) * i, per, bufs[i].ctypes.data, per)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: None, range(threads * 4)))   # start the workers outside the window
        t0 = time.perf_counter()
        list(ex.map(work, range(threads)))
        wall = time.perf_counter() - t0
    total = per * threads
    if w.nkeys > 1:
        shape = f"{threads} threads x {rows} key rows x {w.n} counters (the workload's row shape)"
    else:
        shape = f"{threads} threads x {per} consecutive counters (disjoint shards of the workload's counter range)"
    return total / wall, total, wall, shape


def one_core_rates(key: int, window: int = 1 << 24, reps: int = 5) -> dict:
    """the oracle on ONE core, a `window`-sample run per kind, median of
    `reps`, in Msamples/s, each with a dead-code guard computed from its output after the timed
    call (XOR-fold of the outputs; fused: the histogram total)."""
    import numpy as np

    import oracle as O
    lib = O.lib()
    M64 = (1 << 64) - 1
    kv = np.array([key & M64], dtype=np.uint64)
    res = {}
    for kind in ("u32", "u64", "f32", "fused", "u32_xorfold"):
        ts, guard = [], 0
        if kind in ("u32", "u64", "f32"):
            buf = np.empty(window, dtype={"u32": np.uint32, "u64": np.uint64, "f32": np.uint32}[kind])
            buf.fill(0)
        for r in range(reps):
            c0 = r * window
            if kind == "fused":
                h, o = np.zeros(65536, np.uint64), np.zeros(32, np.uint64)
                t0 = time.perf_counter()
                lib.oracle_fused_stats(key & M64, c0, window, h.ctypes.data, o.ctypes.data)
                ts.append(time.perf_counter() - t0)
                guard ^= int(h.sum()) ^ int(o[0])
            elif kind == "u32_xorfold":
                t0 = time.perf_counter()
                g = lib.oracle_xorfold_u32(key & M64, c0, window)
                ts.append(time.perf_counter() - t0)
                guard ^= int(g)
            else:
                fn = getattr(lib, f"oracle_fill_{kind}")
                t0 = time.perf_counter()
                fn(kv.ctypes.data, 1, c0, window, buf.ctypes.data, window)
                ts.append(time.perf_counter() - t0)
                guard ^= int(np.bitwise_xor.reduce(buf.view(np.uint64 if kind == "u64" else np.uint32)))
        res[kind] = {"msamples_per_s": window / statistics.median(ts) / 1e6, "guard": f"{guard:#x}"}
    return {"window": window, "reps": reps, "statistic": "median", "rates": res,
            "note": "one thread; u32/u64/f32 write a buffer (XOR of it printed as the guard), "
                    "u32_xorfold writes nothing (its fold is the result), fused counts hist + ones"}


def cpu_baseline_line(w: SI.Workload, budget_s: float, one_core: bool = True) -> dict:
    """The cpu_baseline object (both arms build it with this function on the same workload)."""
    cores = host_cores()
    keys = _oracle_keys(w, min(w.nkeys, 64))
    runs = sorted((oracle_rate(w, keys[0], keys, budget_s, cores) for _ in range(3)), key=lambda r: r[0])
    rate, samples, wall, shape = runs[1]   # the median of three runs
    out = {"value": rate / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
           "cpu_model": cpu_model(),
           "sample": f"{samples} samples of {w.name}: {shape}; {wall:.2f} s wall (median of 3 runs: "
                     + ", ".join(f"{r[0] / 1e9:.2f}" for r in runs) + " Gsamples/s)"}
    if one_core:
        out["one_core"] = one_core_rates(keys[0])
    return out


# ------------------------------------------------------------------------------------- GPU arm
def run_ours(args, w: SI.Workload, rank: int, world: int, dev: int, entry: str = "auto"):
    """Times `args.steps` steps of workload w on this rank.  entry: "auto" = the by-value
    entry point sq_fill_*_k for single-key fills (key in the launch parameters), "devkeys" =
    the 8(b) call sq_fill_* with a device key array."""
    import torch
    import torch.distributed as tdist

    import paper_2004_06278_b200 as sq
    from paper_2004_06278_b200 import dist as sqdist

    if args.scaling == "weak":
        # weak scaling (opt-in; per-GPU work fixed): rank r owns the r-th config-sized block of
        # the counter space -- or the r-th block of nkeys keys -- so N GPUs do N batches.
        if w.shard == "key":
            keys_all = sq.keygen(w.key_seed, w.nkeys * world)
            k0, kn = rank * w.nkeys, w.nkeys
            ctr0, n = w.ctr0, w.n
        else:
            keys_all = sq.keygen(w.key_seed, 1)
            k0, kn = 0, 1
            ctr0, n = (w.ctr0 + rank * w.n) & ((1 << 64) - 1), w.n
    else:
        # strong scaling (default; BASELINE.json's configs split a fixed total): the config's
        # counters (c2, c3, c5) or key rows (c4) in contiguous shards
        keys_all = sq.keygen(w.key_seed, w.nkeys)
        if w.shard == "key":
            k0, kn = sqdist.key_shard(w.nkeys)
            ctr0, n = w.ctr0, w.n
        else:
            k0, kn = 0, 1
            ctr0, n = sqdist.counter_shard(w.ctr0, w.n)
    key0 = int(keys_all[k0]) & ((1 << 64) - 1)
    keys_d = keys_all[k0:k0 + kn].cuda(dev)
    samples_rank = kn * n
    stream = torch.cuda.current_stream(dev)
    if w.kind == "fused":
        # hist and ones are the two views of ONE packed buffer: zeroed by one memset, exchanged
        # by one in-place all-reduce
        buf, hist, ones = sqdist.counts_buffer(dev)

        def step():
            # one pass of the whole path over one batch: counts from zero,
            # generate-and-reduce, and at N > 1 the one all-reduce of the counts (same stream)
            buf.zero_()
            sq.fused_stats(key0, ctr0, n, hist, ones, stream=stream)
            if world > 1:
                sqdist.allreduce_counts(hist, ones)
    else:
        out = torch.empty((kn, n), dtype={"u32": torch.int32, "u64": torch.int64, "f32": torch.float32}[w.kind],
                          device=dev)
        if kn == 1 and entry == "auto":
            # single key: the by-value entry point (sq_fill_*_k), key in the launch parameters
            fill_k = getattr(sq, f"fill_{w.kind}_k")
            out1 = out.view(-1)

            def step():
                fill_k(key0, ctr0, n, out=out1, stream=stream)
        else:
            fill = getattr(sq, f"fill_{w.kind}")

            def step():
                fill(keys_d, ctr0, n, out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize(dev)
        if world > 1:
            tdist.barrier()
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            tdist.barrier()
    ms = evs[0].elapsed_time(evs[-1])
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    nb = min(20, args.steps)
    burst_ms = sum(per_step[:nb]) / nb          # the first launches: before the power cap engages
    t = torch.tensor([ms, burst_ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(samples_rank)], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tdist.all_reduce(tot, op=tdist.ReduceOp.SUM)
    ms_max, burst_max = float(t[0].item()), float(t[1].item())
    total_samples = float(tot.item())
    clocks = clk.summary()
    res = {
        "ms_total": ms_max,
        "ms_per_step": ms_max / args.steps,
        "value": total_samples * args.steps / (ms_max * 1e-3) / 1e9,
        "burst": {"value": total_samples / (burst_max * 1e-3) / 1e9, "steps": nb,
                  "ms_per_step": burst_max,
                  "note": f"mean of the first {nb} timed steps (max over ranks); `value` is all {args.steps}"},
        "samples_per_step": int(total_samples),
        "samples_rank": samples_rank,
        "clocks": clocks,
        "key0": key0,
        "kn": kn,
    }
    if world > 1:
        allc = [None] * world
        tdist.all_gather_object(allc, {"rank": rank, "sm_mhz": clocks.get("sm_mhz"), "reasons": clocks.get("reasons"),
                                       "ms": ms, "samples": samples_rank})
        res["per_rank"] = allc
    if w.kind == "fused" and world > 1:   # the exchange alone (it is also inside every timed step)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            sqdist.allreduce_counts(hist, ones)
        e1.record()
        torch.cuda.synchronize(dev)
        res["allreduce_ms"] = e0.elapsed_time(e1) / 10
    # e2e through the C ABI with host buffers (rank-local shard)
    if not args.no_e2e:
        res["e2e"] = run_e2e(args, w, sq, key0, keys_d, ctr0, n, kn, dev, world)
    return res


def run_e2e(args, w, sq, key0, keys_d, ctr0, n, kn, dev, world):
    import torch
    import torch.distributed as tdist
    steps = args.e2e_steps
    if w.kind == "fused":
        from paper_2004_06278_b200 import dist as sqdist
        host = torch.empty(65536 + 32, dtype=torch.int64).pin_memory()
        buf, hist, ones = sqdist.counts_buffer(dev)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(steps):
            buf.zero_()
            sq.fused_stats(key0, ctr0, n, hist, ones)
            if world > 1:
                sqdist.allreduce_counts(hist, ones)
            host.copy_(buf, non_blocking=True)
            torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        d2h = (65536 + 32) * 8
        samples = n
    else:
        es = 8 if w.kind == "u64" else 4
        rows = [int(k) & ((1 << 64) - 1) for k in keys_d[: min(kn, 8)].tolist()] if w.shard == "key" else [key0]
        # key-sharded workloads: time the first min(kn, 8) rows of this rank, scale by rows
        host = torch.empty(n * es * len(rows), dtype=torch.uint8).pin_memory()
        scratch = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
        cs = torch.cuda.Stream(dev)
        sq.fill_host(w.kind, rows[0], ctr0, min(n, 1 << 20), host, scratch, copy_stream=cs)  # warm
        t0 = time.perf_counter()
        for _ in range(steps):
            for i, k in enumerate(rows):
                sq.fill_host(w.kind, k, ctr0, n, host[i * n * es:(i + 1) * n * es], scratch, copy_stream=cs)
        wall = time.perf_counter() - t0
        d2h = n * es * len(rows)
        samples = n * len(rows)
    t = torch.tensor([wall], dtype=torch.float64, device=dev)
    s = torch.tensor([float(samples)], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tdist.all_reduce(s, op=tdist.ReduceOp.SUM)
    return {"value": float(s.item()) * steps / float(t.item()) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": 8, "d2h_bytes_per_step": d2h, "steps": steps,
            "d2h_GBps": d2h * steps / float(t.item()) / 1e9 if world == 1 else None,
            "note": "sq_fill_host (chunked generate + D2H into pinned memory) / fused_stats (+ the all-reduce at "
                    "N > 1) + D2H of the counts; host wall clock, max over ranks; the 8-byte key travels in the "
                    "launch parameters"}


def config_for(w: SI.Workload, world: int, scaling: str) -> dict:
    """The `config` object of the JSON line -- identical for both arms (ours and --impl reference)."""
    per_rank = w.nkeys * w.n
    return {"workload": f"{w.name}: " + {
        "c2": "squares32 fill, 1 key (seed 1), ctr 0..2^30-1, uint32 out (4 GiB)",
        "c3": "squares64 fill, 1 key (seed 1), ctr 0..2^29-1, uint64 out (4 GiB)",
        "c4": "squares32->f32 fill, 4096 keys (seed 7) x 2^18 ctr, [key][ctr] (4 GiB)",
        "c5": "fused squares32 hist(65536)+ones(32), 1 key (seed 1), ctr 0..2^38-1"}[w.name],
        "key_seed": w.key_seed, "nkeys": w.nkeys, "ctr0": w.ctr0, "n_per_key": w.n,
        "samples_per_step": per_rank * world if scaling == "weak" else per_rank,
        "sharding": "counter" if w.shard == "ctr" else "key",
        "parallelism": f"{'ctr' if w.shard == 'ctr' else 'key'}-shard x{world}",
        "l2": "output larger than L2 (4 GiB written per step)" if w.kind != "fused"
        else "no HBM traffic (fused, counts only)"}


def sass_per_sample():
    """SASS instructions and FMA-pipe slots per output sample of each hot loop of the LOADED
    library (cuobjdump; tools/sass_counts.py), or {} if cuobjdump is unavailable."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import sass_counts
        import paper_2004_06278_b200 as sq
        return sass_counts.per_workload(sq.LIB_PATH)
    except Exception as e:  # pragma: no cover
        return {"error": str(e)[:200]}


def roofline_for(w: SI.Workload, res, peaks, peaks_src, prof, sass=None, name=None):
    """Roofline of the dominant (only) kernel of the step."""
    ms_launch = res["ms_per_step"]
    sass = sass or {}
    name = name or w.name
    if w.kind == "fused":
        # ALU/FMA-bound: peak derived in DESIGN.md from the measured IMAD rate (64 lane-results
        # per clock per SM) and the 9 FMA-pipe slots squares32 needs per sample after the
        # finite-difference round 1: 64/9 samples/clk/SM x 148 SMs x max SM clock.
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 64.0 / 9.0 * SM_PER_GPU * mhz * 1e6 / 1e9
        achieved = res["samples_rank"] / (ms_launch * 1e-3) / 1e9
        out = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gsamples/s",
               "frac": achieved / peak, "traffic": None,
               "peak_note": "FMA-pipe floor 9 slots/sample (3 IMAD.WIDE x2 + 3 IMAD) at 64 slots/clk/SM, max SM clock",
               "frac_of_12_slot_ceiling": achieved / (64.0 / 12.0 * SM_PER_GPU * mhz * 1e-3),
               "ceiling_12_slot_note": "SURVEY.md 8(d): 12 IMAD slots/sample (no finite-difference round 1)"}
        out.update(_pipes(prof, w.name, prof.get(w.name, {}).get("kernel", "fused_ws_kernel")
                          if str(prof.get(w.name, {}).get("kernel", "")).startswith("fused") else "fused_ws_kernel"))
        if name in sass:
            out["sass"] = sass[name]
            out["imad_issue"] = _imad_issue(achieved, sass[name], mhz, 3)
        return out
    bytes_launch = res["samples_rank"] * w.elem_bytes
    achieved = bytes_launch / (ms_launch * 1e-3) / 1e9
    peak = float(peaks["hbm_gbs"])
    traffic = None
    kname = {"u32": "fill_kernel<0>", "u64": "fill_kernel<1>", "f32": "fill_kernel<2>"}[w.kind]
    if prof.get(w.name, {}).get("kernel") == kname and w.name in prof:
        traffic = prof[w.name].get("dram_bytes_per_launch")
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_src}, copy read+write)",
           "algorithmic_bytes_per_launch": bytes_launch}
    out.update(_pipes(prof, w.name, kname))
    # the same achieved rate against the other write ceilings SURVEY.md 8(d) names (context only)
    out["other_peaks"] = {"spec_8000_GBps": achieved / 8000.0,
                          "memset_7354_GBps (profiles/r01_microbench_writes.json)": achieved / 7354.4,
                          "sm_store_6327_GBps (STG.256, same file)": achieved / 6326.5}
    if name in sass:
        out["sass"] = sass[name]
        out["imad_issue"] = _imad_issue(res["samples_rank"] / (ms_launch * 1e-3) / 1e9, sass[name],
                                        peaks.get("sm_max_mhz", 1965.0), 4 if w.kind == "u64" else 3)
    return out


def _imad_issue(gsps, sass, mhz, wide):
    """SURVEY.md 8(d)'s "% IMAD peak": samples/s x FMA-heavy slots per sample (from the SASS of
    the hot loop) / (SMs x 64 lane-slots per clock x clock), with IMAD.WIDE/HI weighted 2 (their
    issue cost) and 2.5 (their measured cost in dependent chains); `wide` = WIDE/HI
    instructions per sample."""
    slots = sass.get("fma_slots_per_sample")
    if slots is None:
        return None
    cap = SM_PER_GPU * 64 * mhz * 1e6   # wide: IMAD.WIDE/HI per sample (3 squares32, 4 squares64)
    return {"fma_slots_per_sample": slots, "frac_wide_2": gsps * 1e9 * slots / cap,
            "frac_wide_2p5": gsps * 1e9 * (slots + 0.5 * wide) / cap,
            "note": "achieved x SASS FMA-heavy slots / (148 SMs x 64 x max SM clock)"}


def _pipes(prof, name, kname):
    """Pipe utilisation of the same kernel from the committed ncu capture (profiles/): what binds
    when the HBM fraction is below 1 (the u32/f32 fills are IMAD+ALU-bound)."""
    p = prof.get(name, {})
    if p.get("kernel") != kname:
        return {}
    return {"pipes_ncu": {"fmaheavy_pct": p.get("fmaheavy_pct"), "alu_pct": p.get("alu_pct"),
                          "issue_pct": p.get("issue_active_pct"),
                          "inst_executed_per_sample": p.get("inst_executed_per_sample"),
                          "source": "profiles/ncu_summary.json (ncu --set full, same kernel)"}}


DTYPE = {"u32": "u32", "u64": "u64", "f32": "u32->f32", "fused": "u32"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the config's fixed total split over the ranks (BASELINE.json "
                         "configs); weak: every rank runs one config-sized batch of its own counter block")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary c3/c4/c5 summary")
    ap.add_argument("--cpu-budget", type=float, default=1.0, help="seconds per oracle thread (cpu_baseline)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = SI.CONFIGS[args.workload]

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return main_reference(args, w, rank, world)

    import torch
    import torch.distributed as tdist
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink/NVSwitch; SQ_BENCH_BACKEND=gloo only to exercise the multi-rank logic
        # with several ranks on one GPU (no collective on the fill data path either way)
        backend = os.environ.get("SQ_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
    peaks, peaks_src = load_peaks()
    prof = load_profile_summary()
    import paper_2004_06278_b200 as sq  # noqa: F401  (loads libsquares.so; raises if missing)

    res = run_ours(args, w, rank, world, local)
    extra = {}
    sass = sass_per_sample() if rank == 0 else {}
    if not args.no_extra and args.workload == "c2":
        a2 = argparse.Namespace(**vars(args))
        a2.no_e2e = True
        for name, wname, steps, entry in (("c2_devkeys", "c2", 50, "devkeys"), ("c3", "c3", 20, "auto"),
                                          ("c4", "c4", 20, "auto"), ("c5", "c5", 3, "auto")):
            a2.steps, a2.warmup = steps, 3
            ww = SI.CONFIGS[wname]
            # the same starting point for every secondary line: 2 s idle, so that one config's
            # power draw does not carry into the next one's short measurement
            torch.cuda.synchronize(local)
            time.sleep(2.0)
            r = run_ours(a2, ww, rank, world, local, entry=entry)
            rl = roofline_for(ww, r, peaks, peaks_src, prof, sass, name)
            extra[name] = {"value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"], "steps": steps,
                           "roofline": rl, "clocks": r["clocks"], "gpu_launches": steps, "idle_before_s": 2.0}
            if name == "c2_devkeys":
                extra[name]["entry"] = "sq_fill_u32 (device key array, SURVEY.md 8(b))"
            if "allreduce_ms" in r:
                extra[name]["allreduce_ms"] = r["allreduce_ms"]
            if "per_rank" in r:
                extra[name]["per_rank"] = r["per_rank"]

    if rank == 0:
        rl = roofline_for(w, res, peaks, peaks_src, prof, sass)
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": DTYPE[w.kind],
            "data": "synthetic",
            "config": config_for(w, world, args.scaling),
            "roofline": rl,
            "burst": res["burst"],
            "cpu_baseline": cpu_baseline_line(w, args.cpu_budget, one_core=world == 1),
            "clocks": res["clocks"],
            "gpu_launches": args.steps,
            "impl": "ours",
            "entry": "sq_fill_u32_k (key by value)" if w.kind != "fused" and w.nkeys == 1 else
                     ("sq_fill_f32 (device keys)" if w.kind == "f32" else "sq_fused_stats"),
        }
        if "per_rank" in res:
            line["per_rank"] = res["per_rank"]
        if "allreduce_ms" in res:
            line["allreduce_ms"] = res["allreduce_ms"]
        if "e2e" in res:
            line["e2e"] = res["e2e"]
        if extra:
            line["also"] = extra
        print(json.dumps(line))
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def main_reference(args, w, rank, world):
    """Reference arm: the CPU oracle as it stands on the host cores (rank 0 only).  Its keys come
    from the oracle's own key utility: this process never loads the product library."""
    if rank != 0:
        return
    import oracle as O
    O.build()
    cores = host_cores()
    keys = _oracle_keys(w, min(w.nkeys, 64))
    key0 = keys[0]
    # each step a bounded sample sized so that warmup + steps take <= ~120 s
    per_step_budget = max(0.05, min(args.cpu_budget, 120.0 / (args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_rate(w, key0, keys, per_step_budget / 4, cores)
    tot_s, tot_n = 0.0, 0
    last = None
    for _ in range(args.steps):
        rate, samples, wall, shape = oracle_rate(w, key0, keys, per_step_budget, cores)
        tot_s += wall
        tot_n += samples
        last = (samples, shape)
    value = tot_n / tot_s / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": DTYPE[w.kind],
        "data": "synthetic", "impl": "reference",
        "config": config_for(w, world, args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"per step {last[0]} samples: {last[1]}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
