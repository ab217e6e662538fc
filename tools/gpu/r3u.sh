set -x
PGX_LIB=$PWD/exp/libpgx_v13.so timeout 900 python tools/hub_probe.py C4 0,4096,16384,65536,262144 > gpurun_out/r3u.log 2>&1
timeout 600 python tools/probe.py C4 5 > gpurun_out/r3u_cur.log 2>&1
