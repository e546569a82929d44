"""Write profiles/push_deposit_traffic.json from ncu --set full captures of
the mover kernel, one per workload, each tagged with the sha256 of that
kernel's machine code in the library that was captured (_lib.kernel_digest;
bench.py reports `roofline.traffic` only while the loaded library's kernel
has the same code -- any rebuild of the same sources does).

  python scripts/traffic_json.py c2=gpurun_out/mover_c2.ncu-rep c3=gpurun_out/mover_c3.ncu-rep ...
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def read_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    data = rows[2]
    rec = {}
    for m in METRICS + ["Kernel Name"]:
        i = head.index(m)
        v = data[i].replace(",", "")
        if m == "Kernel Name":
            rec["kernel"] = v
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
                 "msecond": 1e3}.get(units[i], 1.0)
        rec[m] = float(v) * scale
    return {"kernel": rec["kernel"], "ncu_duration_us": rec["gpu__time_duration.sum"],
            "dram_bytes_read": rec["dram__bytes_read.sum"], "dram_bytes_write": rec["dram__bytes_write.sum"],
            "dram_bytes_per_launch": rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"],
            "source": path}


def main():
    from paper_2404_10270_b200 import _lib

    with open(_lib.LIB_PATH, "rb") as fh:
        sha = hashlib.sha256(fh.read()).hexdigest()
    wl = {}
    for arg in sys.argv[1:]:
        name, path = arg.split("=", 1)
        rec = read_rep(path)
        short = rec["kernel"].replace("void ", "").split("(")[0]
        rec["kernel_sass_sha256"] = _lib.kernel_digest(_lib.MOVER_SYMBOLS[short])
        wl[name] = rec
    out = {"lib_sha256": sha, "workloads": wl,
           "source": "ncu --set full --clock-control none (cold cache, one launch per workload)"}
    with open(os.path.join(ROOT, "profiles", "push_deposit_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
