"""Per-ABI-call DRAM traffic from an ncu launch list with dram__bytes_{read,write}.sum
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`), summed over
the kernels each call launches, for one step; written to profiles/<name>.json for bench.py's
roofline `traffic` field.

  python tools/traffic.py gpurun_out/launches_tf.csv transformer profiles/r02_traffic_transformer.json
"""
import csv
import json
import sys

# kernel-name prefixes launched by each ABI call, in step order
CALLS = [
    ("gate_topk", ["k_transpose", "k_tc_gemm<32, 0, 0, 0", "k_tc_gemm<48, 0, 0, 0", "k_tc_gemm<64, 0, 0, 0",
                   "k_tc_gemm<128, 0, 0, 0", "k_tc_gemm<256, 0, 0, 0", "k_simt_rows", "k_prefix_alive", "k_beam_topk",
                   "k_topk_exact"]),
    ("dispatch", ["k_weights_hist", "k_scan_chunks", "k_scan_experts", "k_rank", "k_scatter", "k_gather"]),
    ("expert_ffn_fwd", ["k_tile_plan", "k_tc_gemm<256, 0, 0, 1", "k_tc_gemm<256, 0, 0, 2", "k_tc_gemm<128, 0, 0, 1",
                        "k_tc_gemm<128, 0, 0, 2"]),
    ("combine", ["k_combine<"]),
    ("combine_bwd", ["k_combine_bwd"]),
    ("expert_ffn_bwd", ["k_tile_plan", "k_tc_gemm<256, 0, 1", "k_tc_gemm<128, 0, 1", "k_tc_gemm<128, 1, 1, 4",
                        "k_tc_gemm<256, 1, 1, 4", "k_seg_colsum"]),
    ("gate_bwd", ["k_transpose", "k_gate_bwd_dx", "k_tc_gemm<128, 1, 1, 6", "k_tc_gemm<256, 1, 1, 6",
                  "k_gate_reduce", "k_dwg_partial", "k_dwg_reduce"]),
]


def main(path, name, out):
    rows = list(csv.reader(open(path)))
    hdr, kern = None, {}
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = d["ID"]
            if key not in kern:
                kern[key] = {"name": d["Kernel Name"].split("(")[0].replace("void ", "").replace("dmoe::", "")}
                order.append(key)
            kern[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    allk = [kern[k] for k in order]
    gate = ("k_tc_gemm<32, 0, 0, 0", "k_tc_gemm<48, 0, 0, 0", "k_tc_gemm<64, 0, 0, 0", "k_tc_gemm<128, 0, 0, 0",
            "k_tc_gemm<256, 0, 0, 0", "k_simt_rows")
    starts = [j for j in range(len(allk) - 1)
              if allk[j]["name"].startswith("k_transpose") and allk[j + 1]["name"].startswith(gate)]
    seq = allk[starts[-1]:]  # the last full step (gate transpose .. gate backward)
    per_call, i = {}, 0
    for call, prefixes in CALLS:
        tot = {"bytes": 0.0, "us": 0.0, "kernels": []}
        while i < len(seq) and any(seq[i]["name"].startswith(p) for p in prefixes):
            k = seq[i]
            tot["bytes"] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
            tot["us"] += k.get("gpu__time_duration.sum", 0) / 1e3
            tot["kernels"].append(k["name"])
            i += 1
        per_call[call] = tot
    json.dump({"workload": name, "source": path, "per_call": per_call}, open(out, "w"), indent=1)
    for c, v in per_call.items():
        print(f"{c:16s} {v['bytes'] / 1e9:8.3f} GB {v['us']:9.1f} us  {len(v['kernels'])} kernels")


if __name__ == "__main__":
    main(*sys.argv[1:4])
