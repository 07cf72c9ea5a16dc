"""Per-phase DRAM traffic and time of one step from an ncu raw CSV export
(`ncu -i X.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum,...`), for bench.py's roofline `traffic` field:

    python tools/ncu_traffic.py full.csv > profiles/r02/traffic_c2_bf16.json

Kernels are mapped to bench.py's phases by name; a phase that launches a kernel twice per step
with different grids (the W-row gather and the feature normalize) sums the two."""
import collections
import csv
import json
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}


def phase_of(name: str) -> str:
    m = re.search(r"k_gemm[23]<[^0-9]*([0-9])", name)
    if m:
        # k_gemm2 kinds (fast.cu) and k_gemm3 kinds (fast32.cu: 3/4/6 bf16x3 dX/dW, 5 mixed F)
        return {"0": "gemm_logits_softmax", "1": "gemm_dX", "2": "gemm_dW", "3": "gemm_dX",
                "4": "gemm_dW", "5": "gemm_logits_softmax", "6": "gemm_dW"}[m.group(1)]
    for key, ph in (("k_update_rows", "update"), ("k_normalize_rows", "gather_normalize"),
                    ("k_zero_rows", "gather_normalize"), ("k_rowreduce", "softmax_stats"),
                    ("k_fixup", "softmax_stats"), ("k_dx_reduce", "dX_reduce_scatter"),
                    ("k_feature_backward", "feature_backward")):
        if key in name:
            return ph
    return "other"


rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
ix = {k: i for i, k in enumerate(h)}


def val(r, col):
    v = float(r[ix[col]].replace(",", ""))
    return v * UNITS.get(units[ix[col]], 1)


per = collections.OrderedDict()  # (kernel, grid) -> [bytes, us, n]
for r in rows[2:]:
    if len(r) < len(h):
        continue
    key = (r[ix["Kernel Name"]].split("(")[0], r[ix["Grid Size"]] if "Grid Size" in ix else "")
    e = per.setdefault(key, [0.0, 0.0, 0])
    e[0] += val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    e[1] += val(r, "gpu__time_duration.sum")
    e[2] += 1
out, times = collections.OrderedDict(), collections.OrderedDict()
for (k, _g), (byt, us, n) in per.items():
    ph = phase_of(k)
    out[ph] = out.get(ph, 0) + byt / n
    times[ph] = times.get(ph, 0) + us / n
print(json.dumps({**{k: int(v) for k, v in out.items()},
                  "_us_per_launch": {k: round(v, 2) for k, v in times.items()},
                  "_source": sys.argv[1]}, indent=1))
