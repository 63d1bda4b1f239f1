for st in 16 32; do echo "== stage $st"; BATCHFACT_B200_LIB=build_var/lib_st$st.so python tools/time_variants.py 2>&1 | grep "tier=auto" | grep -v serial; done
