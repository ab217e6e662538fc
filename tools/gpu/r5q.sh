timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5q_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r5q_pytest.log
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5q_seg.log 2>&1
