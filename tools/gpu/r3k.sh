set -x
timeout 900 python tools/seg_check.py C2,C5,C3 off shipped > gpurun_out/r3k.log 2>&1
timeout 600 python tools/probe.py C3 5 > gpurun_out/r3k_probe.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider > gpurun_out/r3k_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r3k_pytest.log
