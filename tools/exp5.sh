for T in 69 133 197; do echo "=== T=$T"; TA_LIB=var/lib_trace.so T=$T LINES=120 python tools/attn_trace.py; done
