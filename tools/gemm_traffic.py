"""DRAM traffic of the six grouped-GEMM launches of one N=1 step from an ncu --set full report.

    ncu --set full --clock-control none -k regex:moe_gemm_pair -c 6 -o gpurun_out/gemm_full \
        python tools/step_once.py 1                     # on the GPU box
    python tools/gemm_traffic.py gpurun_out/gemm_full.ncu-rep > profiles/gemm_traffic.json

Algorithmic bytes per launch = operands + output once, for the bench workload (C2, N=1,
R = n*k = 16384 kept rows, E=8, M=1024, H=4096): fwd1 and dH 243 MB (incl. the 1-bit ReLU
mask), fwd2 and dX 235 MB, the two weight gradients 302 MB (f32 dW).  traffic/algorithmic
near 1 means no operand is re-read from HBM.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

MB = 1e6
R, E, M, H = 16384, 8, 1024, 4096
ALG = {  # (kind, major, epi) template args -> algorithmic bytes
    "fwd1": R * M * 2 + E * H * M * 2 + R * H * 2 + R * H // 8,
    "fwd2": R * H * 2 + E * H * M * 2 + R * M * 2,
    "dH": R * M * 2 + E * H * M * 2 + R * H // 8 + R * H * 2,
    "dX": R * H * 2 + E * H * M * 2 + R * M * 2,
    "wgrad": R * M * 2 + R * H * 2 + E * M * H * 4,
}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def main(rep: str) -> int:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    per, alg = [], []
    roles = {"0, 0, 5": "fwd1", "0, 0, 1": "fwd1", "0, 0, 0": "fwd2", "0, 1, 6": "dH", "0, 1, 2": "dH",
             "0, 1, 0": "dX", "1, 1, 3": "wgrad", "1, 1, 4": "wgrad"}
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
        wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
        targs = d["Kernel Name"].split("<256, ", 1)[1].split(">", 1)[0] if "<256, " in d["Kernel Name"] else ""
        role = roles.get(targs, "?")
        per.append({"kernel": d["Kernel Name"][:60], "role": role,
                    "us": float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "ns" else 1.0),
                    "dram_read_MB": rd / MB, "dram_write_MB": wr / MB,
                    "tensor_pipe_pct": float(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"])})
        alg.append(ALG.get(role, 0))
    tot = sum((p["dram_read_MB"] + p["dram_write_MB"]) * MB for p in per)
    res = {
        "source": f"ncu --set full --clock-control none, one fwd+bwd step (tools/step_once.py, N=1, C2), "
                  f"{len(per)} grouped-GEMM launches ({rep.split('/')[-1]})",
        "dram_bytes_per_launch": tot / max(1, len(per)),
        "algorithmic_bytes_per_launch": sum(alg) / max(1, len(alg)),
        "note": "algorithmic = operands + output once (fwd1/dH 243 MB incl. the 1-bit ReLU mask, fwd2/dX 235 MB, "
                "wgrad 302 MB with f32 dW); traffic/algorithmic ~1: no re-read waste",
        "per_launch": per,
    }
    print(json.dumps(res, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
