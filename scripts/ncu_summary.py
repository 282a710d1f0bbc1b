"""Summarise an ncu --set full report of the bound kernel into profiles/.

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_k1 [launch_list.csv]

Writes <out>.md (pipe utilisation, stall reasons, source hotspots) and updates
profiles/ncu_summary.json (dram bytes per launch, read by bench.py as
roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, out = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    rows = ncu_csv(rep, "--page", "raw")
    h, u, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    units = dict(zip(h, u))
    keys = [
        "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    ]
    lines = [f"# ncu summary: {os.path.basename(rep)}", "", "| metric | value | unit |", "|---|---|---|"]
    for k in keys:
        if k in d:
            lines.append(f"| {k} | {d[k]} | {units.get(k, '')} |")
    lines += ["", "## Warp stall reasons (per issued instruction)", "", "| reason | ratio |", "|---|---|"]
    stalls = []
    for name, val in d.items():
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(val), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for val, name in sorted(stalls, reverse=True)[:12]:
        lines.append(f"| {name} | {val:.3f} |")
    # source hotspots
    try:
        src = ncu_csv(rep, "--page", "source", "--print-source=cuda,sass")
        hdr = src[2]
        iex = hdr.index("Instructions Executed")
        per, txt, cur = collections.Counter(), {}, None
        for r in src[3:]:
            if not r:
                continue
            if r[0].strip():
                try:
                    cur = int(r[0])
                    txt[cur] = r[1].strip()[:90]
                except ValueError:
                    pass
            if len(r) > iex and r[2].strip():
                try:
                    per[cur] += int(r[iex] or 0)
                except ValueError:
                    pass
        tot = sum(per.values()) or 1
        lines += ["", "## Source lines by executed instructions (top 25)", "",
                  "| line | share | source |", "|---|---|---|"]
        for ln, c in sorted(per.items(), key=lambda x: -x[1])[:25]:
            lines.append(f"| {ln} | {100 * c / tot:.1f}% | `{txt.get(ln, '')}` |")
    except Exception as e:  # noqa: BLE001
        lines.append(f"\n(source page unavailable: {e})")
    if launches and os.path.exists(launches):
        lines += ["", "## Launch list (ncu --metrics gpu__time_duration.sum, bench.py command)", ""]
        agg = collections.defaultdict(lambda: [0, 0.0])
        with open(launches) as f:
            body = [ln for ln in f if ln.startswith('"')]
        for r in csv.DictReader(io.StringIO("".join(body))):
            if r.get("Metric Name") == "gpu__time_duration.sum":
                name = r["Kernel Name"][:80]
                agg[name][0] += 1
                val = float(r["Metric Value"].replace(",", ""))
                unit = r.get("Metric Unit", "ns")
                agg[name][1] += val * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                                       "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        total = sum(t for _, t in agg.values()) or 1
        lines += ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{name}` | {cnt} | {t:.3f} | {100 * t / total:.1f}% |")
    with open(out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    summ_path = os.path.join(os.path.dirname(out) or ".", "ncu_summary.json")
    summ = {}
    if os.path.exists(summ_path):
        summ = json.load(open(summ_path))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        rd = float(d["dram__bytes_read.sum"]) * scale.get(units["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"]) * scale.get(units["dram__bytes_write.sum"], 1)
        summ["dram_bytes_per_launch"] = rd + wr
    except (KeyError, ValueError):
        pass
    summ["report"] = os.path.basename(rep)
    summ["duration"] = d.get("gpu__time_duration.sum") + " " + units.get("gpu__time_duration.sum", "")
    json.dump(summ, open(summ_path, "w"), indent=1)
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
