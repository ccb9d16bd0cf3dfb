# session 3: vLLM parity incl. overlap, a repeat of the low/mid-load sweep, ncu of a decode-size capture
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3ovl2; mkdir -p $O
( time timeout 1800 python -m pytest tests/test_gpu_vllm.py -x -q -p no:cacheprovider ) > $O/pytest_vllm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:capture_kernel -s 6 -c 1 -o $O/capture_small python scripts/profile_small.py > $O/ncu_small.log 2>&1
summ() { grep '^{' $1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['capture'], d.get('sites'), d.get('overlap'), d['rate_rps'], 'tpot %.3f tok/s %.0f' % (d['tpot_ms_mean'], d['output_tok_s']))
"; }
R=1,4,16
timeout 1500 python scripts/vllm_serving.py --capture off --rates $R --num-requests 96 > $O/v_off.log 2>&1; summ $O/v_off.log > $O/vllm_summary.txt
for s in resid_post resid_post,mlp_act; do
  for ov in "" "--overlap"; do
    tag=${s//,/_}${ov:+_ovl}
    timeout 1500 python scripts/vllm_serving.py --capture on --sites $s $ov --rates $R --num-requests 96 > $O/v_$tag.log 2>&1
    echo "$tag rc=$?" >> $O/vllm_summary.txt; summ $O/v_$tag.log >> $O/vllm_summary.txt
  done
done
echo done
