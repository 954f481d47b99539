# FP64 leaf kernel A/B probes (tools/f64_ab.py): where does the 8 % DMMA idle go?
for v in base noload nofull cw16; do
  ATA_LIB_PATH=_ab/$v.so timeout 300 python tools/f64_ab.py 58 4096 5
done
ATA_DBG=2 ATA_LIB_PATH=_ab/base.so timeout 300 python tools/f64_ab.py 58 4096 5
ATA_LIB_PATH=_ab/base.so timeout 300 python tools/f64_ab.py 148 4096 3
ATA_LIB_PATH=_ab/base.so timeout 300 python tools/f64_ab.py 58 16384 3
