"""dev helper: digest an ncu report -- headline metrics, stall mix, top stalled
SASS lines and per-instruction L2 sector excess for each kernel.
usage: python tools/ncu_digest.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else None
HEAD = ("Duration", "DRAM Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Executed Ipc Active", "L2 Hit Rate", "Elapsed Cycles", "SM Active Cycles",
        "Dynamic Shared Memory Per Block", "Grid Size")


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
names = []
for row in det[1:]:
    d = dict(zip(h, row))
    k = d["Kernel Name"]
    if filt and filt not in k:
        continue
    if k not in names:
        names.append(k)
        print("\n==", k[:90])
    if d["Metric Name"] in HEAD:
        print("  ", d["Metric Name"], "=", d["Metric Value"], d["Metric Unit"])
for k in names:
    base = k.split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    src = run("--page", "source", "--csv", "--print-source", "sass", "-k", base)
    rows = list(csv.reader(io.StringIO(src)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hh = rows[hdr_i]
    data = []
    for r in rows[hdr_i + 1:]:
        if r and r[0] == "Address":  # next kernel instance of the same name
            break
        if len(r) == len(hh):
            data.append(r)
    ix = {c: i for i, c in enumerate(hh)}
    S = lambda c: sum(float(r[ix[c]] or 0) for r in data)
    tot = S("Warp Stall Sampling (All Samples)") or 1
    print(f"\n-- {base}: stall mix (% of {tot:.0f} samples)")
    print("  ", {c.replace("stall_", ""): round(S(c) / tot * 100, 1) for c in hh
                 if c.startswith("stall_") and "Not Issued" not in c and S(c) / tot > 0.01})
    cnt = Counter()
    for r in data:
        op = [o for o in r[ix["Source"]].split() if not o.startswith("@")]
        cnt[op[0].split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
    t = sum(cnt.values())
    print("   inst", t, [(k2, round(v / t * 100, 1)) for k2, v in cnt.most_common(10)])
    top = sorted(data, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:12]
    for r in top:
        print("  ", r[ix["Address"]][-5:], r[ix["Warp Stall Sampling (All Samples)"]],
              "lsb", r[ix["stall_long_sb"]], "ssb", r[ix["stall_short_sb"]], "wait",
              r[ix["stall_wait"]], r[ix["Source"]][:64])
    for r in data:
        sct = r[ix["L2 Theoretical Sectors Global"]]
        if sct and sct != "0":
            print("   mem", r[ix["Source"]][:56], "sectors", sct, "ideal",
                  r[ix["L2 Theoretical Sectors Global Ideal"]], "exec",
                  r[ix["Instructions Executed"]])
