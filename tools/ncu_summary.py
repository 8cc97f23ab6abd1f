"""Summarise ncu raw-page CSV exports (tools/gpu_profile.sh) into
profiles/r1_ncu_final.json (key metrics per launch) and
profiles/agg_traffic_<workload>.json (DRAM bytes per launch of each
aggregation kernel kind, read by bench.py as roofline.traffic), and the
launch-list CSV into profiles/r1_launches_final.txt.
Usage: ncu_summary.py GPURUN_OUT_DIR [ROUND_TAG]"""

import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg."
        "pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
KINDS = ["agg_sub_ring", "agg_ring_epi", "agg_tf_multi", "agg_tf_ring", "agg_ring",
         "agg_bulk", "gat_ring", "gat_bulk"]
WORKLOAD = {"cfg2": "cfg2", "igbgcn": "igb-medium-gcn",
            "igbgat": "igb-medium-gat", "papers": "papers100m-sage-rank0of8"}


def read_raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")][:96]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = f"{r[i]} {units[i]}".strip()
        rb = wb = 0.0
        for k, acc in (("dram__bytes_read.sum", "r"),
                       ("dram__bytes_write.sum", "w")):
            if k in hdr:
                i = hdr.index(k)
                v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                rb, wb = (v, wb) if acc == "r" else (rb, v)
        rec["dram_bytes_total"] = rb + wb
        out.append(rec)
    return out


def kind_of(name):
    for k in KINDS:
        if f"::{k}<" in name or f" {k}<" in name or f"{k}<" in name:
            return k
    return None


def main():
    src = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out")
    tag_round = sys.argv[2] if len(sys.argv) > 2 else "r1"
    final = {"note": "ncu --set full --clock-control none, one bench step "
                     "per workload (tools/gpu_profile.sh), per launch; "
                     "tensor-pipe utilisation of the tcgen05 transforms: "
                     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_"
                     "realtime",
             "kernels": {}}
    for tag, workload in WORKLOAD.items():
        p = src / f"ncu_{tag}_raw.csv"
        if not p.exists():
            continue
        recs = read_raw(p)
        final["kernels"][tag] = recs
        traffic = defaultdict(list)
        for r in recs:
            k = kind_of(r["kernel"])
            if k:
                traffic[k].append(r["dram_bytes_total"])
        if traffic:
            out = {k: sum(v) / len(v) for k, v in traffic.items()}
            out["source"] = (f"profiles/{tag_round}_ncu_final.json: dram__bytes_read."
                             "sum + dram__bytes_write.sum per launch of that "
                             "kernel kind, ncu --set full")
            (ROOT / "profiles" / f"agg_traffic_{workload}.json").write_text(
                json.dumps(out, indent=1))
    (ROOT / "profiles" / f"{tag_round}_ncu_final.json").write_text(
        json.dumps(final, indent=1))
    lp = src / "launches_cfg2.csv"
    if lp.exists():
        rows = [r for r in csv.reader(open(lp)) if len(r) > 5]
        hdr = rows[0]
        ki, mi, vi = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"))
        tot = defaultdict(lambda: [0, 0.0])
        for r in rows[1:]:
            if r[mi] == "gpu__time_duration.sum":
                v = float(r[vi].replace(",", ""))
                unit = r[hdr.index("Metric Unit")]
                ms = v / 1e6 if unit in ("ns", "nsecond") else (
                    v / 1e3 if unit in ("us", "usecond") else v)
                tot[r[ki][:90]][0] += 1
                tot[r[ki][:90]][1] += ms
        allms = sum(t[1] for t in tot.values())
        lines = ["ncu --metrics gpu__time_duration.sum --clock-control none "
                 "-c 400: python bench.py --steps 2 --warmup 1 "
                 "--no-cpu-baseline",
                 "(warmup + 2 timed + 1 metrics step + stable-backend steps "
                 "+ e2e steps; cold-cache, serialised)",
                 "launches  total_ms  share  kernel"]
        for name, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"{n:4d}  {ms:9.3f} ms  {100 * ms / allms:4.1f}% "
                         f"{name}")
        (ROOT / "profiles" / f"{tag_round}_launches_final.txt").write_text(
            "\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
