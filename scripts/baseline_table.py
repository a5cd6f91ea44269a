"""Fill BASELINE.md §4 ("Measured") from the committed evidence: oracle goldens (tests/golden/configs.txt),
1-GPU kernel times (a JSONL from scripts/ab_configs.py) and per-config ncu metric captures
(gpurun_out/ncuq_<cfg>.csv: ncu --metrics ... --csv of one search-kernel launch).

    python scripts/baseline_table.py --times profiles/configs_r2.jsonl --ncu-dir profiles/ncu_r2
"""
import argparse
import csv
import io
import json
import os
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden():
    rows = {}
    for line in open(os.path.join(ROOT, "tests", "golden", "configs.txt")):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            rows[f[0]] = dict(count=int(f[1]), hash=f[2], tasks=int(f[3]), secs=float(f[5]), threads=int(f[6]))
    return rows


def ncu_metrics(path):
    if not os.path.exists(path):
        return {}
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name, unit, val = d.get("Metric Name"), d.get("Metric Unit"), d.get("Metric Value")
        if not name:
            continue
        try:
            v = float(val.replace(",", ""))
        except (ValueError, AttributeError):
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-6,
                 "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)
        out[name] = v * scale
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--times", required=True)
    ap.add_argument("--ncu-dir", required=True)
    a = ap.parse_args()
    gold = golden()
    times = {}
    for line in open(a.times):
        r = json.loads(line)
        times.setdefault(r["config"], []).extend(r["kernel_ms"])
    print("| config | count | hash | oracle threads / wall | 1×B200 kernel ms (median) | bicliques/s (1 GPU) | "
          "HBM GB/s | L2 GB/s | L2 hit | issue active | SIMT lanes | I-cache hit |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for c in ["C2", "C3", "C4", "C5", "C5p"]:
        g = gold.get(c)
        t = times.get(c)
        m = ncu_metrics(os.path.join(a.ncu_dir, f"ncuq_{c}.csv"))
        if not g or not t:
            continue
        med = statistics.median(t)
        dur = m.get("gpu__time_duration.sum")
        dram = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
        l2 = m.get("lts__t_bytes.sum")
        fmt = lambda x, f: f.format(x) if x is not None else "—"  # noqa: E731
        print(f"| {c} | {g['count']:,} | {g['hash']} | {g['threads']} / {g['secs']:.0f} s | {med:.2f} | "
              f"{g['count'] / med * 1e3:.3g} | {fmt(dram / dur / 1e6 if dur else None, '{:.0f}')} | "
              f"{fmt(l2 / dur / 1e6 if (l2 and dur) else None, '{:.0f}')} | "
              f"{fmt(m.get('lts__t_sector_hit_rate.pct'), '{:.1f} %')} | "
              f"{fmt(m.get('smsp__issue_active.avg.pct_of_peak_sustained_active'), '{:.1f} %')} | "
              f"{fmt((m.get('smsp__thread_inst_executed_per_inst_executed.ratio') or 0) / 32 or None, '{:.2f}')} | "
              f"{fmt(m.get('sm__icc_request_hit_rate.pct'), '{:.1f} %')} |")


if __name__ == "__main__":
    main()
