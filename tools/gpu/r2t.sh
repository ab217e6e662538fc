set -x
timeout 900 python tools/seg_check.py C2,C5,C3 shipped > gpurun_out/r2t_seg.log 2>&1; echo "seg rc=$?"
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py -x -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2t_pytest.log
