#!/usr/bin/env python
"""Summarise the ncu captures of profiles/run_profile.sh (gpurun_out/*.ncu-rep)
into profiles/<round>/ncu_summary.json and .md: duration, DRAM bytes per
launch, pipe utilisation, occupancy and the top stall reasons of each hot
kernel. bench.py reads the DRAM bytes as `roofline.traffic`.

    python profiles/summarize_ncu.py gpurun_out profiles/r01
"""
import csv
import io
import json
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "instructions": "smsp__inst_executed.sum",
    "eligible_warps_per_cycle": "smsp__warps_eligible.avg.per_cycle_active",
    "issued_ipc": "smsp__inst_executed.avg.per_cycle_active",
}
# a capture of a hot sweep below these is a gated early-exit launch, not the
# kernel (round 1 committed such a capture): refuse it
MIN_SWEEP = {"duration_us": 20.0, "instructions": 1e6}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ns": 1e-3, "ms": 1e3}


def summarize(rep):
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    # several launches in one report: keep the longest (gated early-exit launches are a few us)
    di = hdr.index("gpu__time_duration.sum")
    data = max(rows[2:], key=lambda r: float(r[di].replace(",", "")) * UNIT_SCALE.get(units[di], 1) if len(r) > di and r[di] else 0.0)
    out = {"kernel": data[hdr.index("Kernel Name")]}
    for key, m in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            v = float(data[i].replace(",", "")) if data[i] else None
            out[key] = v * UNIT_SCALE.get(units[i], 1) if v is not None else None
    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(data[i])
              for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled")
              and h.endswith("_per_issue_active.ratio") and data[i]}
    out["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
    return out


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    res = {}
    for name in ("sweep_points", "sweep_pts1", "sweep_stored", "point_eval"):
        rep = os.path.join(src, name + ".ncu-rep")
        if os.path.exists(rep):
            res[name] = summarize(rep)
            if name.startswith("sweep"):
                bad = [k for k, lo in MIN_SWEEP.items() if (res[name].get(k) or 0.0) < lo]
                if bad:
                    raise SystemExit(f"{rep}: {bad} below the minimum of a real sweep launch "
                                     f"({res[name]}) - a gated launch was captured")
    with open(os.path.join(dst, "ncu_summary.json"), "w") as f:
        json.dump(res, f, indent=2)
    lines = ["| capture | kernel | µs | DRAM read | DRAM write | regs | issue % | XU % | FMA % | warps % | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, v in res.items():
        st = ", ".join(f"{a} {b:.2f}" for a, b in v["top_stalls"].items())
        lines.append(f"| {k} | `{v['kernel'][:48]}` | {v['duration_us']:.1f} | {v['dram_read_bytes'] / 1e6:.2f} MB | "
                     f"{v['dram_write_bytes'] / 1e6:.2f} MB | {v['registers']:.0f} | {v['issue_active_pct']:.1f} | "
                     f"{v['xu_pipe_pct']:.1f} | {v['fma_pipe_pct']:.1f} | {v['warps_active_pct']:.1f} | {st} |")
    with open(os.path.join(dst, "ncu_summary.md"), "w") as f:
        f.write("ncu --set full --clock-control none (one launch each, cold cache; times are not bench "
                "values)\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
