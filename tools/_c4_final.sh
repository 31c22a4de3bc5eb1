# round-2 closing c4 refresh (one B200): full GPU suite, c4 bench line, c4 launch list, smoke
F=gpurun_out/final2; mkdir -p $F
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $F/pytest_gpu.log 2>&1; echo pytest rc $?; tail -1 $F/pytest_gpu.log
timeout 300 python bench.py --workload c4 > $F/bench_c4_n1.json 2> $F/bench_c4.err; echo bench c4 rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/ncu_launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 1 > $F/ncu_launches_c4.log 2>&1; echo ncu launches rc $?
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo smoke rc $?; tail -1 $F/smoke.log
