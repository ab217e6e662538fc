set -x
timeout 900 python tools/seg_check.py C2,C5 off pred=0 pred=1 pred=2 > gpurun_out/r2q_seg.log 2>&1; echo "seg rc=$?"
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py -x -q -p no:cacheprovider > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2q_pytest.log
