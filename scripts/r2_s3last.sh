# session 3 last: shipped build -- smoke, default bench + reference arm, launch list, ncu, serving sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3last; mkdir -p $O
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 1500 python bench.py --steps 20 --warmup 3 ) > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 3 ) > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --legs value > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:capture_kernel -c 4 -o $O/capture_full python scripts/profile_capture.py > $O/ncu_full.log 2>&1
summ() { grep '^{' $1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['capture'], d.get('sites'), d.get('overlap'), d['rate_rps'], 'tpot %.3f tok/s %.0f' % (d['tpot_ms_mean'], d['output_tok_s']))
"; }
R=1,4,16,64
timeout 1500 python scripts/vllm_serving.py --capture off --rates $R --num-requests 128 > $O/v_off.log 2>&1; summ $O/v_off.log > $O/vllm_summary.txt
for s in resid_post resid_post,mlp_act; do
  for ov in "" "--overlap"; do
    tag=${s//,/_}${ov:+_ovl}
    timeout 1500 python scripts/vllm_serving.py --capture on --sites $s $ov --rates $R --num-requests 128 > $O/v_$tag.log 2>&1
    echo "$tag rc=$?" >> $O/vllm_summary.txt; summ $O/v_$tag.log >> $O/vllm_summary.txt
  done
done
echo done
