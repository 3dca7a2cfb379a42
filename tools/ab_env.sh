# A/B of one env switch in the bench context (sweep, power-capped clocks), interleaved.
# usage: bash tools/ab_env.sh VAR valueA valueB [reps]
V=$1; A=$2; B=$3; N=${4:-3}
for i in $(seq $N); do
for x in $A $B; do
env $V=$x python bench.py --no-cpu --no-fp32 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$V=$x', d['value'], d['clocks']['sm_mhz'], ' '.join('%s:%.0f'%(g,v['images_per_s']) for g,v in d['per_gamma'].items()))"
done; done
