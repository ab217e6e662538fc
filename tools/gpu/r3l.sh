set -x
timeout 1500 python -m pytest tests/test_gpu_partitioned.py tests/test_gpu_peer_ipc.py tests/test_bench_contract.py tests/test_gpu_c5.py -x -q -p no:cacheprovider > gpurun_out/r3l.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r3l.log
