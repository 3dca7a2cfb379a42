python -m pytest tests/test_gpu_forward.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_scatter.csv python tools/launch_list.py -8 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ll_scatter.csv -v > gpurun_out/ll_scatter.txt; head -16 gpurun_out/ll_scatter.txt
GAMMAS=-16,-8 python tools/graph_time.py 2>&1 | grep gamma
