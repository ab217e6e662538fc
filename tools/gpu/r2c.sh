set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2c_pytest.log
timeout 900 python tools/seg_check.py C2,C5 512,256,128,64 > gpurun_out/r2c_seg.log 2>&1; echo "seg rc=$?"
