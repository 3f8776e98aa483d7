bash scripts/ab_cfg3.sh 2 --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline
bash scripts/ab_cfg3.sh 2 --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline
bash scripts/ab_cfg3.sh 2
