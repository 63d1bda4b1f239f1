for v in base new base new; do echo "== $v"; BATCHFACT_B200_LIB=build_var/lib_$v.so python tools/time_variants.py 2>&1 | grep "tier=auto" | grep -v serial | grep -v "32x32"; done
