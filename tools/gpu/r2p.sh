set -x
timeout 900 python bench.py > gpurun_out/r2p_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2p_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2p_launches.csv python bench.py --steps 2 --warmup 3 --no-per-config --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2p_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2p_ncu_c5 python tools/probe.py C5 1 > gpurun_out/r2p_ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2p_ncu_c2 python tools/probe.py C2 1 > gpurun_out/r2p_ncu_c2.log 2>&1; echo "ncu3 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pagerank_pull_kernel -c 1 -o gpurun_out/r2p_ncu_c4 python tools/probe.py C4 1 > gpurun_out/r2p_ncu_c4.log 2>&1; echo "ncu4 rc=$?"
