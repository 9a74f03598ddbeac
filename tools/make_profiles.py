"""Copy one tools/profile_round.sh run (gpurun_out/prof) into the tracked profiles/ directory.

  python tools/make_profiles.py [--src gpurun_out/prof] [--round r01]

Writes profiles/<round>_bench_<cfg>.json (the bench JSON line), <round>_launches_C1.csv,
<round>_ncu_<capture>_summary.json (key metrics of each --set full capture) and
traffic_<cfg>.json (DRAM bytes per launch of the forward / backward kernel, which bench.py
copies into roofline.traffic). A direction without a capture in this run keeps its previous
figure and says so.
"""
import argparse
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

# capture name per (config, direction)
CAPTURES = {
    "C1": ("C1_fwd", "C1_bwd"), "C2": ("C2_tile", "C2_bwd"), "C3": ("C3_fwd", "C3_bwd"),
    "C4": ("C4_tc", "C4_apply"), "C5": ("C5_fwd", "C5_bwd"), "M1": ("M1_fwd", "M1_bwd"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out", "prof"))
    ap.add_argument("--round", default="r01")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    a = ap.parse_args()
    out = a.out
    os.makedirs(out, exist_ok=True)
    if out != os.path.join(ROOT, "profiles"):  # previous traffic figures for directions not captured
        for f in glob.glob(os.path.join(ROOT, "profiles", "traffic_*.json")):
            dst = os.path.join(out, os.path.basename(f))
            if not os.path.exists(dst):
                shutil.copy(f, dst)
    for f in sorted(glob.glob(os.path.join(a.src, "bench_*.json"))):
        cfg = os.path.basename(f)[6:-5]
        lines = [x for x in open(f).read().splitlines() if x.strip().startswith("{")]
        if lines:
            open(os.path.join(out, f"{a.round}_bench_{cfg}.json"), "w").write(lines[-1] + "\n")
    lc = os.path.join(a.src, "launches_C1.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(out, f"{a.round}_launches_C1.csv"))
    summaries = {}
    for rep in sorted(glob.glob(os.path.join(a.src, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        dst = os.path.join(out, f"{a.round}_ncu_{name}_summary.json")
        ncu_summary.main(rep, dst)
        summaries[name] = json.load(open(dst))
    for cfg, (fwd, bwd) in CAPTURES.items():
        path = os.path.join(out, f"traffic_{cfg}.json")
        old = json.load(open(path)) if os.path.exists(path) else {}
        t = {"source": f"ncu --set full --clock-control none (cold-cache replay, one launch), round {a.round} "
                       f"(profiles/{a.round}_ncu_*_summary.json); dram__bytes_read.sum + dram__bytes_write.sum "
                       "per launch (bytes)"}
        for key, cap in (("forward", fwd), ("backward", bwd)):
            s = summaries.get(cap)
            if s:
                k = s[0]
                scale = {"[byte]": 1, "[Kbyte]": 1e3, "[Mbyte]": 1e6, "[Gbyte]": 1e9}

                def metric(prefix):
                    name = next(kk for kk in k if kk.startswith(prefix))
                    return float(k[name]) * scale.get(name.split(" ")[-1], 1)

                t[key] = int(round(metric("dram__bytes_read.sum") + metric("dram__bytes_write.sum")))
                t[key + "_kernel"] = k.get("Kernel Name")
            elif key in old:
                t[key] = old[key]
                t[key + "_kernel"] = old.get(key + "_kernel")
                t[key + "_note"] = "not captured this run: previous figure kept"
        if len(t) > 1:
            json.dump(t, open(path, "w"), indent=1)
    print("profiles updated from", a.src)


if __name__ == "__main__":
    main()
