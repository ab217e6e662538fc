set -x
timeout 900 python tools/seg_check.py C2,C5 off shipped > gpurun_out/r2i_seg.log 2>&1; echo "seg rc=$?"
timeout 1500 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2i_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2i_ncu_c5_s0 python tools/cap_probe.py C5 1 > gpurun_out/r2i_ncu_s0.log 2>&1; echo "ncu rc=$?"
