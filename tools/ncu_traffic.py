"""Turn an ncu metrics CSV of the persistent MINRES kernel into the traffic
record bench.py reads (profiles/r02_minres_traffic_<workload>.json).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:minres_kernel -s <warm-up launches> -c <launches of one step> \
      --csv --log-file gpurun_out/traffic_c4.csv python tools/minres_profile.py c4
  python tools/ncu_traffic.py c4 gpurun_out/traffic_c4.csv <ic0_mode> [note]

One bench step = the workload's solves (one launch each); the record holds
the launches of ONE step and their DRAM byte sum, the commit the capture was
taken on and the IC(0) apply mode of the profiled kernel variant.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
        "nsecond": 1.0}


def parse(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    by_id = {}
    for r in rows:
        d = by_id.setdefault(r["ID"], {"kernel": r["Kernel Name"]})
        val = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        d[r["Metric Name"]] = val
    return [by_id[k] for k in sorted(by_id, key=int)]


def main():
    import bench
    tag, path, mode = sys.argv[1], sys.argv[2], sys.argv[3]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    launches = [{"kernel": d["kernel"][:60], "dram_read": int(d["dram__bytes_read.sum"]),
                 "dram_write": int(d["dram__bytes_write.sum"]), "ns": int(d["gpu__time_duration.sum"])}
                for d in parse(path)]
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                            text=True).stdout.strip()
    rec = {"workload": bench.WORKLOADS[tag]["label"], "ic0_mode": mode, "commit": commit,
           "kernel": "minres_kernel (persistent, cooperative; one launch = one MINRES solve)",
           "source": os.path.basename(path), "launches": launches,
           "dram_bytes_per_step": sum(l["dram_read"] + l["dram_write"] for l in launches), "note": note}
    out = os.path.join(ROOT, "profiles", f"r02_minres_traffic_{tag}.json")
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(out, rec["dram_bytes_per_step"])


if __name__ == "__main__":
    main()
