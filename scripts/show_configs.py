"""Print run_configs.py JSON lines compactly (kernel ms, phase shares)."""
import json
import sys

NAMES = ["root", "list", "bitrow", "steal", "idle", "popwait", "Lp", "rscan", "cls", "order", "lbuild", "chk", "exp",
         "Qord", "cbuild", "prune"]
for f in sys.argv[1:]:
    print("==", f)
    for line in open(f):
        try:
            d = json.loads(line)
        except ValueError:
            print(line.strip()[:200])
            continue
        ph = " ".join(f"{n}={v:.3f}" for n, v in zip(NAMES, d.get("phase_frac_of_warp_time", [])) if v > 0.005)
        print(d["config"], d["count"], d["tasks"], [round(x, 2) for x in d["kernel_ms"]], "frames", d.get("frames"),
              "maxtask", d.get("max_task_ms"), "roots_out", d.get("roots_out_ms"), "|", ph)
