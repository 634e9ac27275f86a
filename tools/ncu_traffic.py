"""Per-kernel-class launch list of one step from `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv` (tools/profile_step.py): launches, serialised
time, share of the step and DRAM bytes per class (the library's hps_kernel_stats classes).

usage: python tools/ncu_traffic.py launches.csv [CONFIG_KEY out.json]
  prints the table; with CONFIG_KEY (e.g. C4) merges {class: {avg_dram_bytes_per_launch, ...}}
  into out.json (profiles/ncu_traffic.json, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import sys

CLASSES = [  # (substring of the kernel name, class) -- first match wins
    ("zgemv", "zgemv"), ("zgemm_kernel", "zgemm_dmma"), ("zsplit_reduce", "zgemm_dmma"), ("zgj_seq_kernel", "leaf_gj"), ("zgj_ws_kernel", "leaf_gj"),
    ("dgj_leaf_kernel", "leaf_gj"), ("leaf_real_ops_kernel", "leaf_gj"), ("zgj_panel", "zgj_panel"),
    ("zgj_small", "zgj_small"), ("zgj_fused", "zgj_fused"), ("nat_block_inv", "zgj_panel"), ("nat_diag", "zgj_aux"),
    ("zgj_", "zgj_aux"),
    ("leaf_schur_assemble", "leaf_assemble"), ("leaf_assemble", "leaf_assemble"), ("zcopy", "layout"),
    ("rhs_", "layout"), ("zsum_slots", "layout"), ("c_bounds", "leaf_assemble"), ("leaf_R", "layout"),
]


def klass(name):
    for key, c in CLASSES:
        if key in name:
            return c
    return "other"


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h = rows[0]
    ii, ik, im, iv = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"name": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    return list(launches.values())


def summarise(launches):
    agg = collections.defaultdict(lambda: {"launches": 0, "ns": 0.0, "dram": 0.0})
    for d in launches:
        a = agg[klass(d["name"])]
        a["launches"] += 1
        a["ns"] += d.get("gpu__time_duration.sum", 0.0)
        a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ns"] for a in agg.values())
    return agg, tot


def per_kernel(launches):
    """Per kernel name (template arguments kept): launches, serialised time, DRAM bytes."""
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in launches:
        k = d["name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += d.get("gpu__time_duration.sum", 0.0)
        agg[k][2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, (n, ns, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{ns / 1e6:10.3f} ms {100 * ns / tot:5.1f}% {n:6d} launches {by / 1e9:10.2f} GB "
                   f"{by / max(ns, 1) / 1e3:5.1f} TB/s  {k}")
    out.append(f"{tot / 1e6:.3f} ms total, {sum(a[0] for a in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    L = load(sys.argv[1])
    if len(sys.argv) > 2 and sys.argv[2] == "--kernels":
        print(per_kernel(L))
        sys.exit(0)
    agg, tot = summarise(L)
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        print(f"{k:14s} {a['launches']:6d} launches {a['ns'] / 1e6:10.3f} ms {100 * a['ns'] / tot:5.1f}%  "
              f"DRAM {a['dram'] / 1e9:8.2f} GB  {a['dram'] / max(a['launches'], 1) / 1e6:9.2f} MB/launch")
    print(f"total {len(L)} launches, {tot / 1e6:.3f} ms serialised (cold-cache, ncu)")
    if len(sys.argv) > 3:
        key, out = sys.argv[2], sys.argv[3]
        try:
            tab = json.load(open(out))
        except Exception:
            tab = {}
        tab[key] = {k: {"avg_dram_bytes_per_launch": round(a["dram"] / max(a["launches"], 1)),
                        "launches_per_step": a["launches"], "serialised_ms": round(a["ns"] / 1e6, 3),
                        "share_of_step": round(a["ns"] / tot, 4), "dram_bytes_per_step": a["dram"]}
                    for k, a in agg.items()}
        tab["_note"] = ("per kernel class over every launch of one step captured by ncu --metrics "
                        "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                        "(tools/profile_step.py; tools/ncu_traffic.py); times are serialised and cold-cache")
        json.dump(tab, open(out, "w"), indent=1)
