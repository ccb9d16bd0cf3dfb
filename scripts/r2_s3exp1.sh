# session 3: fixes check, ring-full stall repro, meta-ring A/B (device vs host-mapped)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3exp1; mkdir -p $O
( time timeout 900 python -m pytest tests/test_gpu_replicas.py tests/test_gpu_observer.py -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
for v in product hostmeta; do
  if [ $v = product ]; then unset TF_LIB_VARIANT; else export TF_LIB_VARIANT=$v; fi
  timeout 150 python scripts/exp_bigwait.py --n 24 --timeout 90 > $O/bigwait_$v.log 2>&1; echo "rc=$?" >> $O/bigwait_$v.log
  for busy in "" "--busy-d2h"; do
    tag=$v${busy:+_busy}
    timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128 --row-bytes 8192 $busy --out $O/dec128_$tag.json > $O/dec128_$tag.log 2>&1
    timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 448 --row-bytes 28672 $busy --out $O/dec448_$tag.json > $O/dec448_$tag.log 2>&1
    timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 32768,114688 --row-bytes 8192 $busy --out $O/big_$tag.json > $O/big_$tag.log 2>&1
  done
done
unset TF_LIB_VARIANT
echo done
