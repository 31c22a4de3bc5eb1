# round-2 closing measurements (one B200): GPU suite, bench lines, c4 launch list, ncu captures
# exported to CSV on the box (the .ncu-rep files are ~22 MB each and are not brought back)
F=gpurun_out/final; mkdir -p $F
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $F/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $F/pytest_gpu.log 2>&1; echo pytest rc $?; tail -2 $F/pytest_gpu.log
for w in c4 c3 c1 c2 c0; do
  timeout 600 python bench.py --workload $w > $F/bench_${w}_n1.json 2> $F/bench_${w}.err; echo bench $w rc $?
done
DDQD_LU_TRSM=blk timeout 300 python bench.py --workload c4 > $F/bench_c4_trsm_blk.json 2>/dev/null; echo trsm_blk rc $?
DDQD_LU_SPLIT=0 DDQD_LU_TRSM=blk timeout 300 python bench.py --workload c4 > $F/bench_c4_coop_blk.json 2>/dev/null; echo coop rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/ncu_launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 1 > $F/ncu_launches_c4.log 2>&1; echo ncu launches rc $?
for k in lu_subdiag lu_subbelow lu_subgemm; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o /tmp/ncu_full_$k python bench.py --workload c4 --steps 1 --warmup 0 > $F/ncu_full_$k.log 2>&1; echo ncu $k rc $?
  ncu -i /tmp/ncu_full_$k.ncu-rep --page raw --csv > $F/ncu_full_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu_full_$k.ncu-rep --page details --csv > $F/ncu_full_${k}_details.csv 2>/dev/null
done
du -sh $F
