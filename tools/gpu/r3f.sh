set -x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3f_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r3f_pytest.log
timeout 900 python bench.py > gpurun_out/r3f_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r3f_ref.log 2>&1; echo "ref rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r3f_ncu_c5 python tools/probe.py C5 1 > gpurun_out/r3f_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3f_launches.csv python bench.py --steps 2 --warmup 3 --no-per-config --no-cpu-baseline --e2e-steps 1 > gpurun_out/r3f_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
