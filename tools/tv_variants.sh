BATCHFACT_B200_LIB=build_var/lib_new.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "svd or rsvd" 2>&1 | tail -1
for v in base new base new; do echo "== $v"; BATCHFACT_B200_LIB=build_var/lib_$v.so python tools/time_variants.py 2>&1 | grep "tier=auto" | grep "V=1" | grep -v serial; done
