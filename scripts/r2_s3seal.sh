# session 3: sealed completion (TF_CAP_SEALED) -- all gpu tests, sweeps sealed vs per-CTA bytes, bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3seal; mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
for sl in "" "--sealed"; do
  for busy in "" "--busy-d2h"; do
    tag=$([ -n "$sl" ] && echo sealed || echo flags)${busy:+_busy}
    timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 $sl $busy --reps 7 --out $O/dec_$tag.json > $O/dec_$tag.log 2>&1
    timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 1024,32768,114688 --row-bytes 8192 $sl $busy --reps 7 --out $O/big_$tag.json > $O/big_$tag.log 2>&1
  done
done
( time timeout 1500 python bench.py --steps 20 --warmup 3 --legs value,e2e,model ) > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
echo done
