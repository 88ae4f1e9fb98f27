# Round-end evidence on one B200 (run under gpurun from the repo root):
# GPU tests, smoke, the bench line, the ncu launch list of the bench command, and full ncu
# captures of the batched kernel, the cluster learning kernel and the encoder.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sp_batched -s 3 -c 1 -o gpurun_out/prof_batched python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --learn-frames 0 --no-encoder > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sp_learn_cluster -s 1 -c 1 -o gpurun_out/prof_learn python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-learn-full --no-encoder > gpurun_out/ncu_learn.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o gpurun_out/prof_encode python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-learn-full --learn-frames 0 > gpurun_out/ncu_enc.log 2>&1; echo ncu4=$?
tail -3 gpurun_out/gpu_tests.log
cat gpurun_out/smoke.log
