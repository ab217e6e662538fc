set -x
timeout 900 python tools/seg_check.py C2,C5 off shipped shipped > gpurun_out/r2z_seg.log 2>&1; echo "seg rc=$?"
nvidia-smi --query-gpu=clocks.sm,clocks.mem,temperature.gpu,power.draw --format=csv
