# A/B of the fused proj+merge path in the bench context (sweep, power-capped clocks), interleaved
for i in 1 2 3; do
for f in 0 1; do
TA_MERGE_FUSION=$f python bench.py --no-cpu --no-fp32 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('fusion=$f', d['value'], d['clocks']['sm_mhz'], ' '.join('%s:%.0f'%(g,v['images_per_s']) for g,v in d['per_gamma'].items()))"
done; done
