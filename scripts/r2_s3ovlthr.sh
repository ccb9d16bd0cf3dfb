# session 3: overlap with a size threshold (small captures forked, large inline)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3ovlthr; mkdir -p $O
( time timeout 1500 python -m pytest tests/test_gpu_observer.py tests/test_gpu_vllm.py -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
summ() { grep '^{' $1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['capture'], d.get('sites'), d.get('overlap'), d.get('overlap_max_kib'), d['rate_rps'], 'tpot %.3f tok/s %.0f' % (d['tpot_ms_mean'], d['output_tok_s']))
"; }
R=1,4,16,64
timeout 1500 python scripts/vllm_serving.py --capture off --rates $R --num-requests 128 > $O/v_off.log 2>&1; summ $O/v_off.log > $O/vllm_summary.txt
for s in resid_post resid_post,mlp_act; do
  for ov in "" "--overlap --overlap-max-kib 512"; do
    tag=${s//,/_}${ov:+_thr}
    timeout 1500 python scripts/vllm_serving.py --capture on --sites $s $ov --rates $R --num-requests 128 > $O/v_$tag.log 2>&1
    echo "$tag rc=$?" >> $O/vllm_summary.txt; summ $O/v_$tag.log >> $O/vllm_summary.txt
  done
done
echo done
