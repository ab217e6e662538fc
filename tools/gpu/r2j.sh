set -x
timeout 900 python tools/seg_check.py C2,C5 off shipped > gpurun_out/r2j_seg.log 2>&1; echo "seg rc=$?"
timeout 900 python tools/pr_seg_probe.py C4 12 13 > gpurun_out/r2j_prseg.log 2>&1; echo "prseg rc=$?"
timeout 1500 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2j_pytest.log
