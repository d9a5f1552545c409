#!/bin/bash
# GEMM pipeline depth: 6 (in-tree), 5 and 4 stages, ncu-locked-clock A/B of the fused FFN launches
out=gpurun_out/st; mkdir -p $out
L='"" tools/probes/variants/nodeps.so "" tools/probes/variants/nodeps.so'
eval timeout 900 ncu --metrics gpu__time_duration.sum -k regex:moe_gemm --csv --log-file $out/ab_base.csv \
  python tools/probes/ffn_ncu_ab.py 10 $L > $out/ab_base.log 2>&1; echo "ncu base rc=$?"
eval python tools/probes/ffn_ncu_ab.py --parse $out/ab_base.csv 10 $L
