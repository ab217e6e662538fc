for r in 1 2; do
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5g_cur_$r.log 2>&1
for v in vs2 vs4; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5g_${v}_$r.log 2>&1; done
done
