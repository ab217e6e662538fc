set -x
timeout 900 ncu --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r3n_s0 python tools/cap_probe.py C5 1 > gpurun_out/r3n.log 2>&1; echo "rc=$?"
