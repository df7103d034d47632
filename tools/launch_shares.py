"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import io
import re
import sys


def main(path, out, header="one full C2 LF build (tools/one_step.py between cudaProfilerStart/Stop)"):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                  "msecond": 1.0}.get(unit, 1e-6)
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("hf::", "")
        tot[name] += ms
        cnt[name] += 1
    total = sum(tot.values())
    with open(out, "w") as f:
        f.write("# ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none\n")
        f.write(f"# {header}; per-launch times are cold-cache and serialised\n")
        f.write(f"# total {total:.2f} ms over {sum(cnt.values())} launches\n")
        f.write("kernel,launches,total_ms,share_pct,avg_us\n")
        for k in sorted(tot, key=tot.get, reverse=True):
            f.write(f"{k},{cnt[k]},{tot[k]:.3f},{100 * tot[k] / total:.2f},{1000 * tot[k] / cnt[k]:.2f}\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
