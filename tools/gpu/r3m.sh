set -x
for mk in 0x7FFFFF 0x1FFFFF 0x3FFFFFF; do
PGX_LIB=$PWD/exp/libpgx_sv$mk.so timeout 900 python tools/seg_check.py C5 shipped > gpurun_out/r3m_$mk.log 2>&1
done
