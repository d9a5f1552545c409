#!/bin/bash
out=gpurun_out/bit; mkdir -p $out
timeout 600 python tools/probes/bitident.py tools/probes/variants/prev.so > $out/bitident.log 2>&1; echo "bitident rc=$?"; tail -6 $out/bitident.log
