set -x
timeout 300 python tools/ride_ab.py bound 2>&1 | grep prods
for v in bulk_NOSTORE bulk_NOADD; do
ATA_LIB_PATH=_ab/$v.so timeout 300 python tools/ride_ab.py bound 2>&1 | grep prods
done
