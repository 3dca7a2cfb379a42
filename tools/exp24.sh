for g in -8 -16; do echo "gamma $g"; TA_LIB=var/lib_mtrace.so GAMMA=$g python tools/match_trace.py; done
