"""profiles/traffic.json from ncu --set full captures of the PCG kernels
(tools/refresh_profiles.sh ncu): dram__bytes_read.sum + dram__bytes_write.sum per
launch, averaged per kernel; k_update_pxring = (7 k_update_p + 1 k_update_xring) / 8
(the ring's round mix), the key bench.py's roofline line reads.

    python tools/make_traffic.py c2=gpurun_out/r02_pcg_c2.ncu-rep c5=gpurun_out/r02_pcg_c5.ncu-rep
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def per_kernel(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    acc = collections.defaultdict(list)
    for d in data:
        m = re.search(r"(k_\w+)<(\d+)(?:,\s*(\d+))?>", d[ix["Kernel Name"]])
        if not m or (m.group(3) not in (None, "0")):
            continue  # the SpMM's residual mode (check path) is not part of a round
        b = sum(float(d[ix[k]]) * UNIT.get(units[ix[k]], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        acc[f"{m.group(1)}<{m.group(2)}>"].append(b)
    res = {k: int(sum(v) / len(v)) for k, v in acc.items()}
    for kp in {k.split("<")[1] for k in res}:
        p, x = res.get(f"k_update_p<{kp}"), res.get(f"k_update_xring<{kp}")
        if p and x:
            res[f"k_update_pxring<{kp}"] = int((7 * p + x) / 8)
    return res


def main(args):
    out = {}
    for a in args:
        cfg, path = a.split("=", 1)
        out[cfg] = per_kernel(path)
    out["_source"] = ("ncu --set full --clock-control none, tools/profile_pcg.py (one 8-round x-deferral cycle), "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch; "
                      "k_update_pxring = (7 k_update_p + 1 k_update_xring) / 8")
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
