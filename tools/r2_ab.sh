set -u
out=gpurun_out/ab; mkdir -p $out
timeout 300 python tools/probes/kbench.py > $out/kbench.txt 2>&1; echo "kbench rc=$?"; head -2 $out/kbench.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --csv -k regex:moe_gemm_pair --log-file $out/gemm_ncu_ab.csv python tools/probes/gemm_ab.py --eager tools/probes/variants/old.so "" > $out/gemm_ncu_ab.log 2>&1; echo "ncu ab rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
