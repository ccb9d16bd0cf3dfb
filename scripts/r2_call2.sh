cd $GRAFT_REPO_ROOT
LEG_TIMEOUT=420 bash scripts/r2_bench_legs.sh
bash scripts/r2_exp.sh
