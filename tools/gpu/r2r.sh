set -x
timeout 900 python bench.py --steps 10 --no-per-config --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2r_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --config C2 --steps 10 --no-per-config --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2r_c2.log 2>&1; echo "c2 rc=$?"
