"""Summarise ncu outputs into profiles/ (text, committed).

    python tools/summarize_ncu.py launches gpurun_out/launches_r01.csv profiles/r01_launches
    python tools/summarize_ncu.py full gpurun_out/sweep_c1_r01.ncu-rep profiles/r01_sweep_c1 --bytes 6432000000
"""
import csv
import json
import subprocess
import sys

SCALE_MS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
            "s": 1e3, "second": 1e3}

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def launches(src, out):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    per = {}
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        ms = float(r[vi].replace(",", "")) * SCALE_MS.get(r[ui], 1.0)
        name = r[ki]
        per.setdefault(name, []).append(ms)
        seq.append((name, ms))
    total = sum(ms for _, ms in seq)
    with open(out + ".md", "w") as fh:
        fh.write(f"# launch list ({src})\n\n`ncu --metrics gpu__time_duration.sum --clock-control none` "
                 "(cold-cache, serialised: compare shares, not absolutes)\n\n")
        fh.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            fh.write(f"| `{name[:60]}` | {len(v)} | {sum(v):.3f} | {sum(v) / total:.4f} |\n")
        fh.write("\n## sequence\n\n| # | kernel | ms |\n|---|---|---|\n")
        for i, (name, ms) in enumerate(seq):
            fh.write(f"| {i} | `{name[:40]}` | {ms:.4f} |\n")
    print(open(out + ".md").read()[:2000])


def full(rep, out, alg_bytes):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, h in enumerate(hdr):
        if h in KEYS:
            d[h] = {"value": vals[i], "unit": units[i]}
    t_ms = float(d["gpu__time_duration.sum"]["value"].replace(",", "")) * SCALE_MS.get(
        d["gpu__time_duration.sum"]["unit"], 1.0)
    rd = float(d["dram__bytes_read.sum"]["value"].replace(",", "")) * (
        1e9 if d["dram__bytes_read.sum"]["unit"] == "Gbyte" else 1e6 if d["dram__bytes_read.sum"]["unit"] == "Mbyte" else 1)
    wr = float(d["dram__bytes_write.sum"]["value"].replace(",", "")) * (
        1e9 if d["dram__bytes_write.sum"]["unit"] == "Gbyte" else 1e6 if d["dram__bytes_write.sum"]["unit"] == "Mbyte" else 1)
    summ = {"report": rep, "kernel": "rapdb_solver_kernel OP_PROBE (one fused C1 sweep: packed-symmetric stream + unit-partial reduction + g combine + U copy-out)",
            "duration_ms": t_ms, "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_sweep": rd + wr, "algorithmic_bytes_per_sweep": alg_bytes,
            "traffic_over_algorithmic": (rd + wr) / alg_bytes if alg_bytes else None,
            "achieved_gbs_algorithmic": alg_bytes / (t_ms / 1e3) / 1e9 if alg_bytes else None,
            "metrics": d}
    json.dump(summ, open(out + ".json", "w"), indent=1)
    src = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(out + "_details.csv", "w").write(src)
    print(json.dumps({k: v for k, v in summ.items() if k != "metrics"}, indent=1))


MULTI = KEYS + ["lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts.sum",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors.sum",
                "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
                "smsp__cycles_active.avg", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
                "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "launch__occupancy_limit_registers",
                "sm__warps_active.avg.per_cycle_active"]


def multi(rep, out):
    """One row per captured kernel launch (a report with several kernels)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    res = []
    for vals in rows[2:]:
        if len(vals) <= ki:
            continue
        d = {"kernel": vals[ki]}
        for i, h in enumerate(hdr):
            if h in MULTI and i < len(vals):
                d[h] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    json.dump(res, open(out + ".json", "w"), indent=1)
    for d in res:
        print(d["kernel"][:50], d.get("gpu__time_duration.sum"), d.get("dram__bytes_read.sum"),
              d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
              d.get("l1tex__data_pipe_lsu_wavefronts.sum"))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "multi":
        multi(sys.argv[2], sys.argv[3])
    else:
        ab = float(sys.argv[sys.argv.index("--bytes") + 1]) if "--bytes" in sys.argv else 0.0
        full(sys.argv[2], sys.argv[3], ab)
