timeout 900 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r4g_ncu_c3bu python tools/probe.py C3 1 > gpurun_out/r4g_ncu.log 2>&1; echo "ncu rc=$?"
