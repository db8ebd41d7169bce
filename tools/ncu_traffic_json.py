"""profiles/ncu_traffic.json + profiles/r01_ncu_full_summary.md from the cold
`ncu --set full` captures of tools/gpu/ncu_traffic.sh (gpurun_out/ncu_cold/*.raw.csv).
usage: python tools/ncu_traffic_json.py [round]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCOPE = {"k_l2": "bwd.node_w2grad", "k_l3": "bwd.node_w1grad", "k_l6": "bwd.edge_w2grad", "k_l10": "bwd.edge_w1ab_grad",
         "k_l7": "bwd.edge_dz1_gemm", "k_msg": "fwd.edge_msg_gemm", "k_agg": "fwd.agg_segsum",
         "k_seg": "bwd.segsum_dst_src", "k_a1": "fwd.edge_act", "k_prep": "bwd.edge_act", "k_col": "bwd.colsum_tail",
         "k_fchain": "fwd.node_chain", "k_bchain": "bwd.node_chain", "k_fdx": "bwd.force_edge_dx",
         "k_fgrad": "bwd.force_edge_wgrad", "k_force": "fwd.force_edge_gemm", "k_af0": "fwd.force_act"}


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = os.path.join(ROOT, "gpurun_out", "ncu_cold")
    traffic, rows = {}, []
    for k, scope in SCOPE.items():
        f = os.path.join(src, f"{k}.raw.csv")
        if not os.path.exists(f):
            continue
        r = list(csv.reader(open(f)))
        if len(r) < 3:
            continue
        d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))

        def num(key, scale_to=None):
            v = float(d[key].replace(",", ""))
            unit = u.get(key, "")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
                    "nsecond": 1e-3, "msecond": 1e3}.get(unit, 1)
            return v * mult
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        us = num("gpu__time_duration.sum")
        traffic[scope] = int(rd + wr)
        rows.append((scope, d.get("Kernel Name", "")[:48], us, rd / 1e6, wr / 1e6, (rd + wr) / (us * 1e-6) / 1e9,
                     d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "")))
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch: ncu --set full (default cache control: "
                        "L2 flushed before each pass), one instance per kernel inside a graph replay of the bench step; "
                        "tools/gpu/ncu_traffic.sh")
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    with open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_full_summary.md"), "w") as f:
        f.write("<!-- ncu --set full --clock-control none (cold L2), one instance of each kernel in a graph replay of "
                "the bench step (tools/gpu/ncu_traffic.sh); raw CSVs not committed -->\n\n")
        f.write("| scope | kernel | us (cold) | DRAM read MB | DRAM write MB | DRAM GB/s | warps active % |\n")
        f.write("|---|---|---:|---:|---:|---:|---:|\n")
        for s, n, us, rd, wr, bw, occ in rows:
            f.write(f"| `{s}` | {n} | {us:.1f} | {rd:.2f} | {wr:.2f} | {bw:.0f} | {occ} |\n")
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
