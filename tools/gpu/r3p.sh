set -x
timeout 1800 python tools/ablation.py r2 3 > gpurun_out/r3p_ablation.log 2>&1; echo "rc=$?"
tail -25 gpurun_out/r3p_ablation.log
