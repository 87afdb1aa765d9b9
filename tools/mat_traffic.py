"""Per-product DRAM traffic of the dominant kernel (the materialization launches of the
grouped GEMM) from an ncu --set full report -> profiles/mat_kernel_traffic.json.

usage: python tools/mat_traffic.py gpurun_out/final_mat.ncu-rep CONFIG "how it was captured"
"""
import csv
import io
import json
import subprocess
import sys

rep, cfg, how = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
units = rows[1]
recs = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def val(r, k):
    u = units[hdr.index(k)]
    x = float(r[k].replace(",", ""))
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0) \
        if "bytes" in k else x


rd = sum(val(r, "dram__bytes_read.sum") for r in recs)
wr = sum(val(r, "dram__bytes_write.sum") for r in recs)
ms = sum(val(r, "gpu__time_duration.sum") for r in recs)
res = {"config": cfg, "kernel": "grouped_gemm_ws_kernel<Ws64> materialization launches",
       "source": how, "launches": len(recs), "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_launch": rd + wr, "per": "product (sum over the product's "
       "materialization launches, like roofline.achieved)", "ncu_ms": ms,
       "tensor_active_pct": [float(r["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"])
                             for r in recs]}
json.dump(res, open("profiles/mat_kernel_traffic.json", "w"), indent=1)
print(res)
