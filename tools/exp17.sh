for T in 197 133; do echo "=== T=$T"; TA_LIB=var/lib_trace.so T=$T LINES=150 python tools/attn_trace.py; done
