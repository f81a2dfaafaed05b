"""Summarises ncu captures into profiles/ (committed evidence).

    python scripts/summarize_ncu.py <full.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_kernels.md (per-kernel duration, DRAM traffic, occupancy, IPC, top stall
reasons from the --set full capture), profiles/<tag>_launches.csv (copy of the
gpu__time_duration launch list of the bench command) and profiles/ncu_traffic.json (DRAM bytes
per launch per bench kernel group, read by bench.py for roofline.traffic)."""
from __future__ import annotations

import csv
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
# kernel -> bench.py kernel group (the event-timed phases of integrateScanDevice)
GROUP = {"k_ingest": "ingest", "k_ingest_tma": "ingest", "k_drift_finalize": "drift", "k_apply_offset": "drift",
         "k_side_prep": "drift", "k_fuse_list": "fusion", "k_jump_grid": "rays",
         "k_sort_rowscan": "sort", "k_sort_scatter": "sort", "k_fuse": "fusion", "k_fuse_heavy": "rays",
         "k_classify": "rays", "k_rays_pass1": "rays", "k_remove": "rays", "k_rays_pass2": "rays", "k_rays_tail": "rays",
         "k_cells": "cells", "k_shift": "shift"}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main(rep, launches, tag):
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    h, units, rows = raw_rows(rep)
    col = {n: i for i, n in enumerate(h)}

    # byte counters in MB whatever unit ncu picked for the column (byte / Kbyte / Mbyte / Gbyte)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}

    def val(r, n):
        try:
            v = float(r[col[n]].replace(",", ""))
        except (KeyError, ValueError):
            return None
        if n.startswith("dram__bytes"):
            v *= scale.get(units[col[n]], 1.0)
        return v

    stall_cols = [n for n in h if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    peaks = ROOT / "MEASURED_PEAKS.json"
    hbm = json.loads(peaks.read_text()).get("hbm_gbs", 6450.3) if peaks.exists() else 6450.3
    lines = [f"# ncu summary ({tag})", "",
             f"Source: `{Path(rep).name}` (`ncu --set full --clock-control none --import-source on`, one GPU). "
             "Per-launch times here are cold-cache and serialised; compare shares, not absolutes.",
             f"HBM % = (dram__bytes_read.sum + dram__bytes_write.sum) / duration against the measured "
             f"{hbm:.0f} GB/s copy peak (MEASURED_PEAKS.json). lanes = smsp__thread_inst_executed_per_inst_executed"
             ".ratio / 32 (SIMT lane efficiency). L2 atomics = lts__t_requests_srcunit_tex_op_atom_dot_alu + _cas + "
             "op_red (requests reaching L2; warp-aggregated atomics count once per warp), their rate, and "
             "lts__d_atomic_input_cycles_active (% of the L2 atomic units' peak). L2 GB/s = lts__t_sectors.sum x 32 B / "
             "duration: all traffic through L2, which is where a frame's intermediates live (126 MB L2).", "",
             "| kernel | duration us | DRAM read MB | DRAM write MB | DRAM GB/s | HBM % | L2 GB/s | occupancy % | IPC | "
             "lanes | regs | L2 atomics | atomics/s | L2 atomic unit % | top stalls (samples) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = defaultdict(list)
    for r in rows:
        k = r[col["Kernel Name"]].split("(")[0].split("::")[-1]
        dur = val(r, "gpu__time_duration.sum")
        rd = val(r, "dram__bytes_read.sum")
        wr = val(r, "dram__bytes_write.sum")
        occ = val(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
        ipc = val(r, "sm__inst_executed.avg.per_cycle_active")
        regs = val(r, "launch__registers_per_thread")
        stalls = sorted(((val(r, n) or 0.0, n.replace("smsp__pcsamp_warps_issue_stalled_", "")) for n in stall_cols),
                        reverse=True)[:3]
        bw = (rd + wr) * 1e6 / (dur * 1e-6) / 1e9 if dur and rd is not None else None
        lanes = (val(r, "smsp__thread_inst_executed_per_inst_executed.ratio") or 0.0) / 32.0
        atom = sum(val(r, n) or 0.0 for n in ("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum",
                                             "lts__t_requests_srcunit_tex_op_atom_dot_cas.sum",
                                             "lts__t_requests_srcunit_tex_op_red.sum"))
        aunit = val(r, "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed") or 0.0
        arate = atom / (dur * 1e-6) if dur else 0.0
        l2 = (val(r, "lts__t_sectors.sum") or 0.0) * 32 / (dur * 1e-6) / 1e9 if dur else 0.0
        lines.append(f"| {k} | {dur:.1f} | {rd:.2f} | {wr:.2f} | {bw:.0f} | {100 * bw / hbm:.1f} | {l2:.0f} | {occ:.1f} | "
                     f"{ipc:.2f} | {lanes:.2f} | {regs:.0f} | {atom:.0f} | {arate:.2e} | {aunit:.1f} | "
                     + ", ".join(f"{n} {v:.0f}" for v, n in stalls) + " |")
        base = k.split("<")[0]  # template instances (k_rays_pass1<0>/<1>)
        if base in GROUP:
            traffic[GROUP[base]].append((rd + wr) * 1e6)
    (prof / f"{tag}_kernels.md").write_text("\n".join(lines) + "\n")
    # per frame: every captured frame launches k_ingest exactly once
    frames = max(1, len(traffic.get("ingest", [])))
    tj = {g: sum(v) / frames for g, v in traffic.items()}
    tj["_source"] = (f"profiles/{tag}_kernels.md (dram__bytes_read.sum + dram__bytes_write.sum summed over "
                     f"the group's launches, per frame; {frames} frame(s) captured)")
    (prof / "ncu_traffic.json").write_text(json.dumps(tj, indent=1) + "\n")
    shutil.copy(launches, prof / f"{tag}_launches.csv")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
