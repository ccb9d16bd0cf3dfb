# round-2 full check: gpu tests, smoke, bench (ours + reference), launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2full}; mkdir -p $O
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 900 python bench.py ) > $O/bench.log 2>&1
( time timeout 600 python bench.py --impl reference ) > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --legs value > $O/ncu_bench.log 2>&1
echo done
