set -x
timeout 900 python tools/seg_check.py C2,C5 off shipped > gpurun_out/r2e_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python tools/seg_check.py C3 off shipped min=0 > gpurun_out/r2e_seg3.log 2>&1; echo "seg3 rc=$?"
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2e_pytest.log
