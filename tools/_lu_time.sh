timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "lu or LU" > gpurun_out/pytest_lu.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_lu.log
timeout 300 python bench.py --workload c4 > gpurun_out/c4_split1.json 2> gpurun_out/c4_split1.err; echo bench rc $?
python -c "import json;d=json.loads(open('gpurun_out/c4_split1.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernel_shares'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lu_sub|lu_snap|lu_trsm_warp|lu_panel_coop" --csv --log-file gpurun_out/ncu_split_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 > gpurun_out/ncu_split_c4.log 2>&1; echo ncu rc $?
