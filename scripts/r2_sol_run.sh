set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2sol
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_sol scripts/exp_sol.cu
/tmp/exp_sol > gpurun_out/r2sol/sol.jsonl 2>&1
python scripts/exp_sweep.py --n 16 --sizes-kb 32768,114688,1024 --row-bytes 8192 --out gpurun_out/r2sol/sweep_resid.json > gpurun_out/r2sol/sweep_resid.log 2>&1
python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128 --row-bytes 8192 --out gpurun_out/r2sol/sweep_dec128.json > gpurun_out/r2sol/sweep_dec128.log 2>&1
python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 448 --row-bytes 28672 --out gpurun_out/r2sol/sweep_dec448.json > gpurun_out/r2sol/sweep_dec448.log 2>&1
python scripts/exp_sweep.py --n 32 --batch 64 --sizes-kb 512,1792 --row-bytes 8192 --out gpurun_out/r2sol/sweep_dec64.json > gpurun_out/r2sol/sweep_dec64.log 2>&1
TF_LIB_VARIANT=trace python scripts/exp_trace.py --n 32 --batch 16 --sizes-kb 128,448 > gpurun_out/r2sol/trace_dec.log 2>&1
TF_LIB_VARIANT=trace python scripts/exp_trace.py --n 16 --batch 8 --rows 512 --sizes-mib 32,112 > gpurun_out/r2sol/trace_big.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv /tmp/exp_sol x > gpurun_out/r2sol/ncu_sol.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python scripts/profile_capture.py > gpurun_out/r2sol/ncu_cap.csv 2>&1
python -m pytest tests/test_gpu_llama_config2.py tests/test_gpu_observer.py -x -q > gpurun_out/r2sol/pytest.log 2>&1
