F=gpurun_out/final; mkdir -p $F
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "lu or LU" > $F/pytest_lu.log 2>&1; echo pytest rc $?; tail -1 $F/pytest_lu.log
timeout 300 python bench.py --workload c4 > $F/bench_c4_n1.json 2> $F/bench_c4.err; echo bench c4 rc $?
DDQD_LU_SUB_OVERLAP=0 timeout 300 python bench.py --workload c4 > $F/bench_c4_no_overlap.json 2>/dev/null; echo nooverlap rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/ncu_launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 1 > $F/ncu_launches_c4.log 2>&1; echo ncu launches rc $?
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo smoke rc $?; tail -2 $F/smoke.log
