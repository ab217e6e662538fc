set -x
timeout 900 python tools/seg_check.py C3 off shipped min=128 min=512 > gpurun_out/r2x_seg3.log 2>&1; echo "seg3 rc=$?"
