# Round-2 evidence on one B200 (run under gpurun from the repo root): GPU tests, smoke, the bench
# line, the ncu launch list of the bench command, full ncu captures of the headline batched
# kernel, the local candidate-pruning launch, the grid full-learning kernel and the encoder.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-packed --no-strong-shards --no-patch > gpurun_out/bench_ncu.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sp_batched -s 3 -c 1 -o gpurun_out/prof_batched python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --learn-frames 0 --no-encoder --no-packed --no-strong-shards --no-patch > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o gpurun_out/prof_encode python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-learn-full --learn-frames 0 --no-packed --no-strong-shards --no-patch > gpurun_out/ncu_enc.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sp_learn_grid_full -c 1 -o gpurun_out/prof_gridfull python scripts/c5_dram.py 64 full > gpurun_out/ncu_gf.log 2>&1; echo ncu4=$?
tail -3 gpurun_out/gpu_tests.log; grep -E "^FAILED" gpurun_out/gpu_tests.log | head; tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])
print(json.dumps(d['local_full_learning'])[:600]); print(json.dumps(d['patch'])[:300]); print(json.dumps(d['encoder'])[:400])"
