export SHAPES="256,69,12,64;256,101,12,64;256,117,12,64;256,133,12,64;256,197,12,64"
echo base; python tools/attn_bench.py
echo kvonce; TA_LIB=var/lib_kvonce.so python tools/attn_bench.py
echo kvqonce; TA_LIB=var/lib_kvqonce.so python tools/attn_bench.py
