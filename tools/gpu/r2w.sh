set -x
for c in 3 4; do
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r2w_cap$c python tools/cap_probe.py C5 $c > gpurun_out/r2w_cap$c.log 2>&1; echo "cap$c rc=$?"
done
timeout 1500 python -m pytest tests/test_gpu_partitioned.py tests/test_gpu_peer_ipc.py tests/test_bench_contract.py -x -q -p no:cacheprovider > gpurun_out/r2w_part.log 2>&1; echo "part rc=$?"
tail -2 gpurun_out/r2w_part.log
