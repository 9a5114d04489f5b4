"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py r01
Reads gpurun_out/<tag>_prof_<cfg>.ncu-rep and gpurun_out/<tag>_launches.csv; writes
profiles/<tag>_ncu_<cfg>_raw.csv (full raw page), profiles/ncu_summary.json (per config: kernel,
duration, DRAM traffic per launch, pipe utilisation, issue, occupancy, top stalls) and
profiles/<tag>_launches.csv (the bench command's launch list) with a share summary.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_write_pct_peak": "dram__bytes_write.sum.pct_of_peak_sustained_elapsed",
    "fmaheavy_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "warps_active_per_smsp": "smsp__warps_active.avg.per_cycle_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_atom_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
}
UNIT_SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e3, "msecond": 1e6,
              "nsecond": 1, "ns": 1, "us": 1e3, "ms": 1e6, "GHz": 1e9, "MHz": 1e6, "Hz": 1, "hz": 1}


def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    return r.stdout


def parse(txt):
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")]}
    for k, m in KEYS.items():
        if m in hdr:
            i = hdr.index(m)
            v = vals[i].replace(",", "")
            try:
                x = float(v) * UNIT_SCALE.get(units[i], 1)
            except ValueError:
                x = v
            out[k] = x
    stalls = {h.split("issue_stalled_")[1].replace("_per_issue_active.ratio", ""): float(vals[i])
              for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
    out["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    if "dram_read_bytes" in out and "dram_write_bytes" in out:
        out["dram_bytes_per_launch"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    summary = {}
    for cfg in ("c2", "c3", "c4", "c5"):
        rep = os.path.join(OUT, f"{tag}_prof_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        txt = raw(rep)
        with open(os.path.join(PROF, f"{tag}_ncu_{cfg}_raw.csv"), "w") as f:
            f.write(txt)
        s = parse(txt)
        kname = s["kernel"]
        import re
        m = re.search(r"fill_kernel<\(?(?:int\))?\s*(\d)", kname)
        s["kernel"] = ("fused_ws_kernel" if "fused_ws" in kname else "fused_kernel") if "fused" in kname else \
            (f"fill_kernel<{m.group(1)}>" if m else kname)
        s["kernel_full"] = kname
        s["source"] = f"profiles/{tag}_ncu_{cfg}_raw.csv (ncu --set full --clock-control none)"
        # executed instructions per output sample (warp instructions x 32 / samples of the launch;
        # tools/profile_all.sh launches c2 2^30, c3 2^29, c4 2^30, c5 2^34 samples)
        ns = {"c2": 1 << 30, "c3": 1 << 29, "c4": 1 << 30, "c5": 1 << 34}[cfg]
        for k in ("inst_executed",):
            if isinstance(s.get(k), float):
                s[k + "_per_sample"] = s[k] * 32 / ns
        summary[cfg] = s
    for suffix, key in (("", "launch_list"), ("_c5", "launch_list_c5")):
        launch_list(tag, suffix, key, summary)
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


def launch_list(tag, suffix, key, summary):
    lpath = os.path.join(OUT, f"{tag}_launches{suffix}.csv")
    if os.path.exists(lpath):
        txt = open(lpath).read()
        with open(os.path.join(PROF, f"{tag}_launches{suffix}.csv"), "w") as f:
            f.write(txt)
        lines = [l for l in txt.splitlines() if l.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        tot, per = 0.0, {}
        for r in rows[1:]:
            t = float(r[vi].replace(",", ""))
            tot += t
            name = "fill_kernel" if "fill_kernel" in r[ki] else \
                (("fused_ws_kernel" if "fused_ws" in r[ki] else "fused_kernel") if "fused" in r[ki] else r[ki][:60])
            per.setdefault(name, [0, 0.0])
            per[name][0] += 1
            per[name][1] += t
        cmd = "bench.py --steps 5 --warmup 3 --no-e2e --no-extra" if not suffix else \
            "bench.py --workload c5 --steps 2 --warmup 3 --no-e2e --no-extra"
        summary[key] = {
            "source": f"profiles/{tag}_launches{suffix}.csv (ncu --metrics gpu__time_duration.sum --clock-control none; {cmd})",
            "kernels": {k: {"launches": v[0], "total_ns": v[1], "share": v[1] / tot} for k, v in per.items()},
        }


if __name__ == "__main__":
    main()
