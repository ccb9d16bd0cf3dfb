# session 3: gpu tests (cast/reduce rewrite, gate), cast/reduce rates, staging-mode A/B
# on the model, two replicas on one GPU, then the default bench + launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3full4; mkdir -p $O
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python scripts/exp_ops.py > $O/ops.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:capture_kernel python scripts/exp_ops.py --ncu > $O/ncu_ops.csv 2>&1
( time timeout 600 python bench.py --legs model --staging mapped --steps 20 ) > $O/model_mapped.log 2>&1
( time timeout 600 python bench.py --legs model --steps 20 ) > $O/model_copyengine.log 2>&1
( time timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --replicas-per-gpu 2 --steps 10 --warmup 3 ) > $O/bench_2replicas.log 2>&1
( time timeout 1200 python bench.py --steps 20 --warmup 3 ) > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
( time timeout 600 python bench.py --impl reference --steps 20 --warmup 3 ) > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --legs value > $O/ncu_bench.log 2>&1
echo done
