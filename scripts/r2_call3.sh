cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c3; mkdir -p $O
( time timeout 420 python bench.py --legs c2 ) > $O/bench_c2.log 2>&1; echo "rc=$?" >> $O/bench_c2.log
( time timeout 300 python bench.py --legs gpt2 ) > $O/bench_gpt2.log 2>&1; echo "rc=$?" >> $O/bench_gpt2.log
( time timeout 600 python bench.py --legs overload ) > $O/bench_overload.log 2>&1; echo "rc=$?" >> $O/bench_overload.log
TF_LIB_VARIANT=trace timeout 300 python scripts/exp_trace.py --n 32 --batch 16 --sizes-kb 128,448 > $O/trace_dec.log 2>&1
TF_LIB_VARIANT=trace timeout 300 python scripts/exp_trace.py --n 16 --batch 8 --rows 512 --sizes-mib 32,112 > $O/trace_big.log 2>&1
( time timeout 600 python -m pytest tests/test_gpu_replicas.py tests/test_native_sink.py -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
timeout 600 python scripts/exp_sink.py --dir $GRAFT_REPO_ROOT/gpurun_out/sink_tmp --gib 8 --threads 4,8,16 --python > $O/sink_disk.jsonl 2>&1
timeout 300 python scripts/exp_sink.py --dir /dev/shm/sink_tmp --gib 8 --threads 4,8,16 > $O/sink_shm.jsonl 2>&1
rm -rf $GRAFT_REPO_ROOT/gpurun_out/sink_tmp /dev/shm/sink_tmp
STRESS_N=1500 timeout 900 bash scripts/sanitize.sh
echo done
