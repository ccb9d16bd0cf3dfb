# validate the device-resident meta ring; A/B against the host-mapped build
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c4; mkdir -p $O
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 900 ) > $O/pytest.log 2>&1
( time timeout 400 python bench.py --legs c2 ) > $O/bench_c2.log 2>&1; echo "rc=$?" >> $O/bench_c2.log
for v in product hostmeta; do
  if [ $v = product ]; then unset TF_LIB_VARIANT; else export TF_LIB_VARIANT=$v; fi
  for busy in "" "--busy-d2h"; do
    tag=$v${busy:+_busy}
    timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128 --row-bytes 8192 $busy --out $O/dec128_$tag.json > $O/dec128_$tag.log 2>&1
    timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 448 --row-bytes 28672 $busy --out $O/dec448_$tag.json > $O/dec448_$tag.log 2>&1
    timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 32768,114688 --row-bytes 8192 $busy --out $O/big_$tag.json > $O/big_$tag.log 2>&1
  done
done
unset TF_LIB_VARIANT
STRESS_N=1500 timeout 900 bash scripts/sanitize.sh
mkdir -p $O/sanitize && cp gpurun_out/sanitize/*.log $O/sanitize/ 2>/dev/null
timeout 300 python scripts/exp_ops.py > $O/ops.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:capture_kernel python scripts/exp_ops.py --ncu > $O/ncu_ops.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:capture_kernel -s 2 -c 2 -o $O/capture_full python scripts/profile_capture.py > $O/ncu_full.log 2>&1
( time timeout 600 python bench.py --legs value,model ) > $O/bench_vm.log 2>&1
echo done
