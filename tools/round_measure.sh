# GPU box: full GPU test suite, the default bench line, configs 2 / 4 bench lines, in-forward
# ncu captures + launch lists (tools/profile_inforward.sh <tag>).
TAG=${1:-r02b}
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/${TAG}_gputest.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --model vit_l16 --gammas=-16,0,16 --no-cpu --no-fp32 > gpurun_out/${TAG}_bench_l16.json 2>/dev/null
python bench.py --model vit_h14 --batch 512 --gammas=-24 --no-cpu --no-fp32 > gpurun_out/${TAG}_bench_h14.json 2>/dev/null
bash tools/profile_inforward.sh $TAG > gpurun_out/${TAG}_profile.log 2>&1
