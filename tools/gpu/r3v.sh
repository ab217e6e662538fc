set -x
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider > gpurun_out/r3v.log 2>&1; echo "rc=$?"
tail -2 gpurun_out/r3v.log
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3v_seg.log 2>&1
