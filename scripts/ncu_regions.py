"""Aggregate an ncu source page (cuda,sass) of mbe_search_kernel by search.cu region.

    python scripts/ncu_regions.py gpurun_out/rep.ncu-rep

Prints, per region of search.cu (function line ranges found by scanning the file for the
region markers below) and per other file, the share of warp stall samples, of no-instruction and
long-scoreboard samples, and of executed warp instructions.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def regions():
    """(first line, name) of every top-level function of search.cu, in file order."""
    out = []
    pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(")
    for i, line in enumerate(open(os.path.join(ROOT, "paper_2401_05039_b200/csrc/search.cu")), 1):
        m = pat.match(line)
        if m:
            out.append((i, m.group(1)))
    return out


def main():
    rep = sys.argv[1]
    txt = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                                  stderr=subprocess.DEVNULL).decode()
    regs = regions()
    agg = collections.defaultdict(lambda: [0, 0, 0, 0])
    cur, hdr = None, None
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr, r))
        try:
            ln = int(r[0])
            s, ni, lsb, ie = (int(d[k]) for k in ("Warp Stall Sampling (All Samples)", "stall_no_inst", "stall_long_sb",
                                                  "Instructions Executed"))
        except (ValueError, KeyError):
            continue
        key = cur
        if cur == "search.cu":
            key = "search.cu:?"
            for first, name in regs:
                if first <= ln:
                    key = f"search.cu:{name}"
        a = agg[key]
        a[0] += s
        a[1] += ni
        a[2] += lsb
        a[3] += ie
    tot = [sum(v[i] for v in agg.values()) or 1 for i in range(4)]
    print(f"{'region':44s} {'samples%':>9s} {'no_inst%':>9s} {'long_sb%':>9s} {'inst%':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if v[0] * 200 < tot[0]:
            continue
        print(f"{k:44s} {100 * v[0] / tot[0]:9.2f} {100 * v[1] / tot[0]:9.2f} {100 * v[2] / tot[0]:9.2f} "
              f"{100 * v[3] / tot[3]:7.2f}")
    print(f"total samples {tot[0]}, no_inst {100 * tot[1] / tot[0]:.1f}%, long_sb {100 * tot[2] / tot[0]:.1f}%, "
          f"warp instructions {tot[3]}")


if __name__ == "__main__":
    main()
