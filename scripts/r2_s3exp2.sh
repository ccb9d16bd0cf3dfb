# session 3: model-leg A/B (device vs host-mapped meta ring) x (2 GiB vs 16 GiB ring); c2 per variant
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3exp2; mkdir -p $O
for v in product hostmeta; do
  if [ $v = product ]; then unset TF_LIB_VARIANT; else export TF_LIB_VARIANT=$v; fi
  for mib in 2048 16384; do
    ( time timeout 400 python bench.py --legs model --steps 20 --model-ring-mib $mib ) > $O/model_${v}_$mib.log 2>&1; echo "rc=$?" >> $O/model_${v}_$mib.log
  done
  ( time timeout 300 python bench.py --legs c2 --c2-decode 16 ) > $O/c2_$v.log 2>&1; echo "rc=$?" >> $O/c2_$v.log
done
unset TF_LIB_VARIANT
echo done
