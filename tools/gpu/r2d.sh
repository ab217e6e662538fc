set -x
timeout 1200 python -m pytest tests/test_gpu_partitioned.py -x -q -p no:cacheprovider > gpurun_out/r2d_part.log 2>&1; echo "part rc=$?"
tail -5 gpurun_out/r2d_part.log
timeout 900 python tools/seg_check.py C2,C5 off gate=0 gate=1 L=14,gate=0 L=14,gate=1 L=12,gate=0 > gpurun_out/r2d_seg.log 2>&1; echo "seg rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2d_ncu_c2 python tools/probe.py C2 1 > gpurun_out/r2d_ncu.log 2>&1; echo "ncu rc=$?"
