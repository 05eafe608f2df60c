"""Write profiles/traffic.json (DRAM bytes per launch of the headline kernel, as
the fast CG launches it) from an ncu launch list, stamped with the hash of the
kernel sources it was captured on (bench.py reports it only while they match).
    python tools/traffic_from_launches.py profiles/r2s_launches_bench.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import algorithmic_bytes, kernel_sources_sha  # noqa: E402

SOURCES = ["apply_mma.cu", "tma.cu", "ring.cuh", "device_util.cuh", "internal.h"]
KERNEL = "bp3_p7_mma_kernel<1, 1, 1>"  # CON, DOT, TMA: the fast CG's operator launch

src = sys.argv[1]
rows = list(csv.reader(open(src)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = {}
for r in rows[start + 1:]:
    if len(r) > iv and KERNEL in r[ik]:
        per.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", ""))
assert per, f"no {KERNEL} launches in {src}"
n = len(per)
rd = sum(v["dram__bytes_read.sum"] for v in per.values()) / n
wr = sum(v["dram__bytes_write.sum"] for v in per.values()) / n
t = sum(v["gpu__time_duration.sum"] for v in per.values()) / n
alg = algorithmic_bytes(3, 7, (66, 66, 66))[0]
out = {
    "bp3_p7_66x66x66": {
        "kernel": "bp3_p7_mma_kernel (CG form: ring nodes as column partials, fused p.Ap; u staged by one TMA "
                  "tensor copy per element from the row-pitched search direction), 12-warp schedule",
        "dram_bytes_per_launch": rd + wr,
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "algorithmic_bytes_per_launch": alg,
        "ncu_duration_ms": t / 1e6,
        "kernel_sources": SOURCES,
        "source_sha256_16": kernel_sources_sha(SOURCES),
        "source": f"{os.path.relpath(src, ROOT)} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  "dram__bytes_write.sum --clock-control none -c 400 python bench.py --steps 3 --warmup 3 "
                  f"--no-sweep --no-cpu-baseline): mean over the {n} CG-form operator launches",
    }
}
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
