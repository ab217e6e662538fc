set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3t_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r3t_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3t_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/r3t_smoke.log
