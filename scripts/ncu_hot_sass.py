"""Rank SASS instructions of an ncu capture by stall samples, with their source line.

    python scripts/ncu_hot_sass.py gpurun_out/prof.ncu-rep [--n 30] [--by stall_long_sb]
"""
import argparse
import collections
import csv
import io
import subprocess


def page(rep, mode):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", f"--print-source={mode}"],
                                  stderr=subprocess.DEVNULL).decode()
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--by", default="Warp Stall Sampling (All Samples)")
    a = ap.parse_args()
    addr2src, cur, hdr, src = {}, None, None, None
    for r in page(a.rep, "cuda,sass"):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr, r))
        if d.get("Address", "-") == "-":
            src = f"{cur}:{r[0]} {r[1].strip()[:70]}"
        else:
            addr2src[d["Address"]] = src
    rows = page(a.rep, "sass")
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1
    print(f"total samples {tot}")
    for d in sorted(data, key=lambda d: -int(d[a.by]))[:a.n]:
        print(f"{100 * int(d[a.by]) / tot:5.2f}%  {d['Source'].strip()[:44]:44s}  {addr2src.get(d['Address'])}")
    # per source line totals
    per = collections.Counter()
    for d in data:
        per[addr2src.get(d["Address"])] += int(d[a.by])
    print("\nper source line:")
    for k, v in per.most_common(a.n):
        print(f"{100 * v / tot:5.2f}%  {k}")


if __name__ == "__main__":
    main()
