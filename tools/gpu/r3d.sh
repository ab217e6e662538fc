set -x
timeout 900 python tools/seg_check.py C2,C5,C3 shipped > gpurun_out/r3d.log 2>&1
