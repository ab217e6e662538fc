PGX_LIB=$PWD/exp/libpgx_t.so timeout 600 python tools/probe.py C3 2 > gpurun_out/r4h_t.log 2>&1
