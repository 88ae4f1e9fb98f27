set -x
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sp_batched -s 3 -c 1 -o gpurun_out/prof_batched python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --learn-frames 0 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sp_learn_cluster -s 2 -c 2 -o gpurun_out/prof_learn python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_learn.log 2>&1; echo ncu3_rc=$?
cat gpurun_out/bench.json
