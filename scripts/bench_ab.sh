# roofline pass of bench.py (value leg) per library variant
for v in ${VARIANTS}; do
  [ "$v" = "product" ] && v=""
  TF_LIB_VARIANT=$v timeout 300 python bench.py --legs value --steps 4 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']
print('${v:-product}', 'frac %.3f avg %.2f us eager %.2f us per-kind %s value %.1f' % (r['frac'], r['avg_launch_us'], r['avg_launch_us_eager_back_to_back'], {k: round(x,1) for k,x in r['per_kind_us_event_pair_each'].items()}, d['value']))"
done
