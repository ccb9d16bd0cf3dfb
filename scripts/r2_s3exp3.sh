# session 3: evidence pass -- sanitizers, cast/reduce rates + ncu, capture ncu --set full,
# decode-size sweeps idle/busy, trace, sink throughput on the box, e2e with a file sink
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3exp3; mkdir -p $O
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
for op in none sink pin empty_cache malloc item; do
  for ds in "" "--default-stream"; do
    timeout 100 python scripts/exp_bigwait.py --n 24 --timeout 60 --host-op $op $ds > $O/bigwait_${op}${ds:+_ds}.log 2>&1; echo "rc=$?" >> $O/bigwait_${op}${ds:+_ds}.log
  done
done
df -h / /dev/shm $GRAFT_REPO_ROOT > $O/df.txt 2>&1; lscpu > $O/lscpu.txt 2>&1; free -g >> $O/df.txt
timeout 300 python scripts/exp_ops.py > $O/ops.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:capture_kernel python scripts/exp_ops.py --ncu > $O/ncu_ops.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:capture_kernel -c 4 -o $O/capture_full python scripts/profile_capture.py > $O/ncu_full.log 2>&1
for busy in "" "--busy-d2h"; do
  tag=${busy:+busy}; tag=${tag:-idle}
  timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 $busy --out $O/dec_$tag.json > $O/dec_$tag.log 2>&1
  timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 1024,32768,114688 --row-bytes 8192 $busy --out $O/big_$tag.json > $O/big_$tag.log 2>&1
done
TF_LIB_VARIANT=trace timeout 300 python scripts/exp_trace.py --n 32 --batch 16 --sizes-kb 128,448 > $O/trace_dec.log 2>&1
TF_LIB_VARIANT=trace timeout 300 python scripts/exp_trace.py --n 16 --batch 8 --rows 512 --sizes-mib 32,112 > $O/trace_big.log 2>&1
timeout 600 python scripts/exp_sink.py --dir $GRAFT_REPO_ROOT/gpurun_out/sink_tmp --gib 8 --threads 4,8,16 --python > $O/sink_disk.jsonl 2>&1
timeout 300 python scripts/exp_sink.py --dir /dev/shm/sink_tmp --gib 8 --threads 4,8,16 > $O/sink_shm.jsonl 2>&1
rm -rf $GRAFT_REPO_ROOT/gpurun_out/sink_tmp /dev/shm/sink_tmp
( time timeout 600 python bench.py --legs value,e2e,e2efile --sink-dir $GRAFT_REPO_ROOT/gpurun_out/e2e_sink --e2e-steps 4 ) > $O/bench_e2efile_disk.log 2>&1
( time timeout 600 python bench.py --legs value,e2efile --sink-dir /dev/shm/e2e_sink --e2e-steps 4 ) > $O/bench_e2efile_shm.log 2>&1
rm -rf $GRAFT_REPO_ROOT/gpurun_out/e2e_sink* /dev/shm/e2e_sink*
STRESS_N=1500 timeout 1200 bash scripts/sanitize.sh
mkdir -p $O/sanitize && cp gpurun_out/sanitize/*.log $O/sanitize/ 2>/dev/null
echo done
