set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2k_ncu_c5_s0 python tools/cap_probe.py C5 1 > gpurun_out/r2k_ncu_s0.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2k_ncu_c2_s0 python tools/cap_probe.py C2 1 > gpurun_out/r2k_ncu_s0c2.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/seg_check.py C3 off shipped min=0 > gpurun_out/r2k_seg3.log 2>&1; echo "seg3 rc=$?"
