set -x
PGX_LIB=$PWD/exp/libpgx_t.so timeout 600 python tools/probe.py C3 2 > gpurun_out/r3z_t.log 2>&1
PGX_LIB=$PWD/exp/libpgx_tu4.so timeout 600 python tools/probe.py C3 2 > gpurun_out/r3z_tu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r3z_ncu_c3bu python tools/probe.py C3 1 > gpurun_out/r3z_ncu.log 2>&1; echo "ncu rc=$?"
