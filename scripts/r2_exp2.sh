# round-2 experiment batch 2: fixed-cost decomposition + speculation variants
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2exp2; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_fixed scripts/exp_fixed.cu
timeout 300 /tmp/exp_fixed > $O/fixed.jsonl 2>&1
for v in product smem0 smem1 abl256; do
  if [ $v = product ]; then export -n TF_LIB_VARIANT; unset TF_LIB_VARIANT; else export TF_LIB_VARIANT=$v; fi
  timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 32768,114688 --row-bytes 8192 --out $O/sweep_big_$v.json > $O/sweep_big_$v.log 2>&1
  timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128 --row-bytes 8192 --out $O/sweep_dec_$v.json > $O/sweep_dec_$v.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:capture_kernel python scripts/profile_capture.py > $O/ncu_$v.csv 2>&1
done
unset TF_LIB_VARIANT
timeout 1200 python -m pytest tests/test_gpu_llama_config2.py tests/test_gpu_observer.py tests/test_gpu_exporter.py -x -q > $O/pytest.log 2>&1
