set -x
nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a_pytest.log
timeout 600 python tools/seg_check.py C2,C3,C5 256,512 > gpurun_out/r2a_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/r2a_bench_c2.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/r2a_bench_c5.log 2>&1; echo "bench5 rc=$?"
