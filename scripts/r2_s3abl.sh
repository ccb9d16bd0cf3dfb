# session 3: decode-size fixed cost per build variant (ablations of the capture kernel)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3abl; mkdir -p $O
for v in product abl1 abl256 smem0 noctl; do
  if [ $v = product ]; then unset TF_LIB_VARIANT; else export TF_LIB_VARIANT=$v; fi
  timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 --reps 7 --out $O/dec_$v.json > $O/dec_$v.log 2>&1
  timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 32768 --row-bytes 8192 --reps 7 --out $O/big_$v.json > $O/big_$v.log 2>&1
done
unset TF_LIB_VARIANT
( time timeout 900 python bench.py --impl reference --steps 10 --warmup 2 ) > $O/bench_ref_allcores.log 2>&1
echo done
