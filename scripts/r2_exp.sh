# round-2 experiment batch: fixed-cost decomposition, speed-of-light copy,
# capture sweeps, sanitizers, vLLM CUDA-graph byte check
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2exp; mkdir -p $O
(df -hT /tmp $GRAFT_REPO_ROOT /dev/shm /root; lsblk -o NAME,SIZE,TYPE,ROTA,MODEL,MOUNTPOINT; cat /proc/meminfo | head -3; nproc; lscpu | head -20; numactl -H) > $O/host_probe.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_fixed scripts/exp_fixed.cu > $O/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_sol scripts/exp_sol.cu >> $O/build.log 2>&1
timeout 300 /tmp/exp_fixed > $O/fixed.jsonl 2>&1
timeout 300 /tmp/exp_sol > $O/sol.jsonl 2>&1
timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 32768,114688,1024 --row-bytes 8192 --out $O/sweep_big.json > $O/sweep_big.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128 --row-bytes 8192 --out $O/sweep_dec128.json > $O/sweep_dec128.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 448 --row-bytes 28672 --out $O/sweep_dec448.json > $O/sweep_dec448.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv /tmp/exp_sol x > $O/ncu_sol.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:capture_kernel python scripts/profile_capture.py > $O/ncu_cap.csv 2>&1
timeout 1500 bash scripts/sanitize.sh
( time timeout 1200 python -m pytest tests/test_gpu_vllm.py -x -q -p no:cacheprovider ) > $O/vllm_pytest.log 2>&1
echo done
