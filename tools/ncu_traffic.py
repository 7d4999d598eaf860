"""dev helper: per-launch DRAM traffic of the hot-path kernels from ncu reports
(dram__bytes_read.sum + dram__bytes_write.sum), merged into
profiles/ncu_traffic.json under the given config key, which bench.py reports
as roofline.traffic.

usage: python tools/ncu_traffic.py CONFIG REPORT.ncu-rep [REPORT ...]
Kernels are classified as spread / fft / gather by name; the FFT figure is
the sum of its passes (one launch each)."""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
STAGES = (("spread", ("k_spread",)), ("gather", ("k_gather",)),
          ("fft", ("k_col", "k_row", "k_single", "k_dstep", "k_bluestein_fix")))


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ix = {k: j for j, k in enumerate(h)}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        b = sum(float(r[ix[m]]) * UNIT[units[ix[m]]]
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        yield name, b


def main():
    cfg, reps = sys.argv[1], sys.argv[2:]
    per = {}
    seen = set()
    for rep in reps:
        for name, b in kernels(rep):
            base = name.split("(")[0].replace("void ", "")
            if "k_gather_spans" in base or base in seen:
                continue  # plan-time helper / a repeated launch of the same kernel
            seen.add(base)
            for stage, keys in STAGES:
                if any(k in base for k in keys):
                    per[stage] = per.get(stage, 0.0) + b
                    break
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                        "ncu_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[f"config{cfg}"] = {k: int(v) for k, v in per.items()}
    data["source"] = ("ncu --set full --clock-control none per kernel (dram__bytes_read.sum + "
                      "dram__bytes_write.sum per launch; fft = sum of its passes); reports "
                      "summarised in profiles/r02/r02w_ncu_summary_config*.txt")
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1)
    print(json.dumps(data[f"config{cfg}"]))


if __name__ == "__main__":
    main()
