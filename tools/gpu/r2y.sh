set -x
timeout 900 python tools/seg_check.py C3,C2,C5 off shipped > gpurun_out/r2y_seg.log 2>&1; echo "seg rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2y_pytest.log
