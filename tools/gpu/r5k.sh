set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5k_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r5k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5k_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r5k_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r5k_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r5k_launches.csv python bench.py --steps 2 --warmup 3 --no-per-config --no-cpu-baseline --e2e-steps 1 > gpurun_out/r5k_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
