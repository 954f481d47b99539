set -x
for v in ride_reg ride_NOLOAD ride_NOSTORE ride_NOADD; do
ATA_LIB_PATH=_ab/$v.so timeout 300 python tools/ride_ab.py bound 2>&1 | grep prods
done
