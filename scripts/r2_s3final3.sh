# session 3 final validation of the shipped build: all gpu tests, smoke, default bench, reference arm, launch list, ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3final3; mkdir -p $O
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 1500 python bench.py --steps 20 --warmup 3 ) > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 3 ) > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --legs value > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:capture_kernel -c 4 -o $O/capture_full python scripts/profile_capture.py > $O/ncu_full.log 2>&1
echo done
