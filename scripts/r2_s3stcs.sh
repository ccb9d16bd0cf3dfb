# session 3: evict-first ring stores (st.global.cs) A/B: isolated sweeps, value leg per-kind, model leg
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3stcs; mkdir -p $O
for v in product stcs; do
  if [ $v = product ]; then unset TF_LIB_VARIANT; else export TF_LIB_VARIANT=$v; fi
  timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 32768,114688 --row-bytes 8192 --sealed --reps 7 --out $O/big_$v.json > $O/big_$v.log 2>&1
  ( time timeout 900 python bench.py --legs value,model --steps 20 ) > $O/bench_$v.log 2>&1
done
unset TF_LIB_VARIANT
echo done
