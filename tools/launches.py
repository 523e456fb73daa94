"""Summarise an ncu --metrics gpu__time_duration.sum CSV: the kernels of the last full step."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
first = sys.argv[2] if len(sys.argv) > 2 else "k_transpose"
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0][:70], float(d["Metric Value"]) / 1000))
# a step starts at the gate's transpose, i.e. a k_transpose followed by a tcgen05 GEMM (the gate
# backward's transpose is followed by k_gate_bwd_dx)
starts = [i for i, o in enumerate(out) if first in o[0] and (first != "k_transpose" or
                                                             (i + 1 < len(out) and "k_tc_gemm" in out[i + 1][0]))]
i0 = starts[-2] if len(starts) > 1 else 0
i1 = starts[-1] if len(starts) > 1 else len(out)
tot = sum(o[1] for o in out[i0:i1])
for name, us in out[i0:i1]:
    print(f"{us:8.1f} us {100 * us / tot:5.1f}%  {name}")
print(f"{tot:8.1f} us total ({i1 - i0} launches)")
