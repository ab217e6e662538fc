for rep in 1 2; do
timeout 600 python tools/probe.py C3 5 > gpurun_out/r4l_bu_$rep.log 2>&1
for v in pf pf3 u3 u4; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 600 python tools/probe.py C3 5 > gpurun_out/r4l_${v}_$rep.log 2>&1; done
done
