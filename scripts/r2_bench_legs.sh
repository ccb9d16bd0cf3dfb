# bench legs one by one, each under its own timeout (find the slow one)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2legs}; mkdir -p $O
for leg in value e2e gpt2 model c2 cpu; do
  ( time timeout ${LEG_TIMEOUT:-600} python bench.py --legs $leg ) > $O/bench_$leg.log 2>&1
  echo "rc=$?" >> $O/bench_$leg.log
done
