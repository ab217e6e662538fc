set -x
timeout 900 python tools/seg_check.py C2,C5 off shipped L=13 > gpurun_out/r2m_seg.log 2>&1; echo "seg rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2m_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2m_bench.log 2>&1; echo "bench rc=$?"
