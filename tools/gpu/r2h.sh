set -x
timeout 900 python tools/seg_check.py C2,C5 off shipped gate=1 > gpurun_out/r2h_seg.log 2>&1; echo "seg rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2h_pytest.log
timeout 900 python tests/analysis/ref_python_probe.py C1:3,C2:1 > gpurun_out/r2h_refpy.log 2>&1; echo "refpy rc=$?"
