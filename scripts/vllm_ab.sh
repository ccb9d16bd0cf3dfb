# configs[3]: vLLM online serving, capture off vs on (one engine per setting)
RATES=${RATES:-1,4,16}
N=${N:-64}
summ() { python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); o = d.get('observer') or {}
    print(d['capture'], d.get('sites'), d['rate_rps'], 'tpot mean %.3f med %.3f p99 %.3f ttft %.1f tok/s %.0f' % (d['tpot_ms_mean'], d['tpot_ms_median'], d['tpot_ms_p99'], d['ttft_ms_median'], d['output_tok_s']), 'host_s %.3f steps %s bytes %s drops %s' % (o.get('host_begin_step_s', 0), o.get('steps'), o.get('bytes'), o.get('drops')))
"; }
for cfg in off ${SITESETS:-resid_post resid_post,mlp_act}; do
  if [ "$cfg" = off ]; then args="--capture off"; tag=off; else args="--capture on --sites $cfg"; tag=on_${cfg//,/_}; fi
  timeout ${VT:-1500} python scripts/vllm_serving.py $args --rates $RATES --num-requests $N > gpurun_out/vllm_$tag.log 2>&1
  echo "$tag rc $?"
  grep '^{' gpurun_out/vllm_$tag.log | summ
done
