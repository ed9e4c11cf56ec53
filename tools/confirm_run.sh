set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r16_gpu_tests.log 2>&1; tail -2 gpurun_out/r16_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r16_smoke.log 2>&1; tail -2 gpurun_out/r16_smoke.log
python bench.py > gpurun_out/r16_c3.json 2> gpurun_out/r16_c3.err; tail -c 300 gpurun_out/r16_c3.json
python bench.py --config C1 --steps 200 --warmup 10 --no-cpu-baseline --no-dropin > gpurun_out/r16_c1.json 2>/dev/null
python bench.py --config C2 --steps 200 --warmup 10 --no-cpu-baseline --no-dropin > gpurun_out/r16_c2.json 2>/dev/null
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r16_c4.json 2>/dev/null
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r16_c5.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r16_ref.json 2>/dev/null; tail -c 300 gpurun_out/r16_ref.json
python tools/shard_probe.py --frames 40 --lanes 2 > gpurun_out/r16_shard.json 2>/dev/null; cat gpurun_out/r16_shard.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r16_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "frame/" -o gpurun_out/r16_frame python tools/profile_frame.py > gpurun_out/r16_ncu.log 2>&1
ls -la gpurun_out | grep r16
