"""Summarise an ncu --set full capture of mbe_search_kernel into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep --config C2 --name r1_c2 [--launches launches.csv]

Writes profiles/<name>.md (key metrics, stall reasons, hottest source lines) and
merges {config: {...}} into profiles/ncu_summary.json (read by bench.py for
roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__icc_request_hit_rate.pct",
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return x * scale


def hot_lines(rep, n=25):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                                  stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr = None, None
    agg, text, lsb = collections.Counter(), {}, collections.Counter()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        d = dict(zip(hdr, r))
        try:
            ln = int(r[0])
        except ValueError:
            continue
        if d.get("Address", "-") != "-":
            continue
        k = (cur, ln)
        text[k] = r[1][:100]
        agg[k] += int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        lsb[k] += int(d.get("stall_long_sb", 0) or 0)
    tot = max(1, sum(agg.values()))
    return [(f"{k[0]}:{k[1]}", 100.0 * v / tot, 100.0 * lsb[k] / tot, text[k]) for k, v in agg.most_common(n)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--config", required=True)
    ap.add_argument("--name", required=True)
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    r = raw(a.rep)
    m = {k: r[k] for k in KEYS if k in r}
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v[0].replace(",", "")))
              for k, v in r.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    stot = max(1, sum(stalls.values()))
    dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    dur_v, dur_u = m["gpu__time_duration.sum"]
    dur_ms = float(dur_v.replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}[dur_u.replace("ms", "msecond").replace("us", "usecond").replace("ns", "nsecond") if len(dur_u) == 2 else dur_u]
    summ = {"kernel": "mbe_search_kernel", "duration_ms_under_ncu": dur_ms, "dram_bytes_per_launch": dram,
            "l2_bytes_per_launch": to_bytes(*m["lts__t_bytes.sum"]) if "lts__t_bytes.sum" in m else None,
            "metrics": {k: f"{v} {u}".strip() for k, (v, u) in m.items()},
            "stall_pct": {k: round(100.0 * v / stot, 2) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v}}
    lines = hot_lines(a.rep)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    jp = os.path.join(ROOT, "profiles", "ncu_summary.json")
    allj = json.load(open(jp)) if os.path.exists(jp) else {}
    summ["name"] = a.name
    allj[a.config] = summ
    json.dump(allj, open(jp, "w"), indent=1)
    md = [f"# ncu --set full: mbe_search_kernel, config {a.config} ({a.name})", "",
          "Captured with `ncu --set full --clock-control none --import-source on -k regex:mbe_search_kernel`",
          "(one launch; ncu serialises and replays, so the duration is not a bench number).", "",
          "| metric | value |", "|---|---|"]
    md += [f"| {k} | {v} |" for k, v in summ["metrics"].items()]
    md += ["", f"DRAM bytes per launch: {dram:.3e}", "", "## Warp stall samples (% of all)", "",
           "| reason | % |", "|---|---|"]
    md += [f"| {k} | {v} |" for k, v in list(summ["stall_pct"].items())[:12]]
    md += ["", "## Hottest source lines (% of stall samples; long-scoreboard share)", "",
           "| line | % samples | % long_sb | source |", "|---|---|---|---|"]
    md += [f"| {l} | {p:.1f} | {q:.1f} | `{t.replace('|', '/')}` |" for l, p, q, t in lines]
    if a.launches and os.path.exists(a.launches):
        md += ["", "## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache serialised)", ""]
        rows = list(csv.reader(open(a.launches)))
        hdr = None
        per = collections.defaultdict(list)
        for row in rows:
            if row and row[0] == "ID":
                hdr = row
                continue
            if hdr and len(row) == len(hdr):
                d = dict(zip(hdr, row))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    per[d["Kernel Name"][:60]].append(float(d["Metric Value"].replace(",", "")))
        tot = sum(sum(v) for v in per.values()) or 1.0
        md += ["| kernel | launches | total | share |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            md += [f"| `{k}` | {len(v)} | {sum(v):.0f} | {100 * sum(v) / tot:.1f}% |"]
    open(os.path.join(ROOT, "profiles", f"{a.name}.md"), "w").write("\n".join(md) + "\n")
    print(json.dumps({k: summ[k] for k in ("duration_ms_under_ncu", "dram_bytes_per_launch")}))


if __name__ == "__main__":
    main()
