set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/ride_ab.py 2>&1 | grep prods
ATA_LIB_PATH=_ab/ride_reg.so timeout 300 python tools/ride_ab.py 2>&1 | grep prods
