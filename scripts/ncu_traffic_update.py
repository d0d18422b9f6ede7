"""Record the DRAM traffic of the collide-stream kernel from an ncu launch capture
in profiles/ncu_traffic.json, keyed by workload, precision, kernel, nodes per
launch and the kernel-source hash (bench.py reports roofline.traffic only for a
matching build; a stale entry reads as null).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      -k regex:k_collide_stream -s 3 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline \
      > gpurun_out/ncu_traffic.csv
  python scripts/ncu_traffic_update.py gpurun_out/ncu_traffic.csv --workload config5-weak-tgv-512^3-per-gpu \
      --precision fp64 --kernel 'k_collide_stream_paper<double>' --nodes 134217728
"""
import argparse
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_ncu(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    vals = {}
    for r in rows:
        if r.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                     "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
            vals[r["Metric Name"]] = v * scale
            vals["kernel_name"] = r.get("Kernel Name")
    return vals


def main():
    import bench

    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--precision", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--nodes", type=int, required=True)
    a = ap.parse_args()
    v = parse_ncu(a.csv)
    dram = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    entries = [e for e in d.get("entries", []) if not (
        e["workload"] == a.workload and e["precision"] == a.precision and e["kernel"] == a.kernel and
        int(e["nodes_per_launch"]) == a.nodes)]
    entries.append({"workload": a.workload, "precision": a.precision, "kernel": a.kernel, "nodes_per_launch": a.nodes,
                    "source_hash": bench.kernel_source_hash(), "dram_bytes_per_launch": dram,
                    "dram_bytes_per_node": dram / a.nodes, "duration_ns": v.get("gpu__time_duration.sum"),
                    "ncu_kernel_name": v.get("kernel_name"),
                    "source": f"{os.path.relpath(a.csv, ROOT)}: ncu dram__bytes_read.sum + dram__bytes_write.sum of "
                              "one launch of the bench command (--clock-control none, cold serialised launch)"})
    json.dump({"entries": entries}, open(path, "w"), indent=1)
    print(json.dumps(entries[-1]))


if __name__ == "__main__":
    main()
