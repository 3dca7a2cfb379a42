python tools/split_streams.py
TA_PDL=0 python tools/split_streams.py
K=4 python tools/split_streams.py
