# caller-layout path: tests, step time, bench line, launch list
set -x
OUT=gpurun_out/cl2
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -k "caller or seam or elements" > $OUT/pytest_cl.log 2>&1; tail -2 $OUT/pytest_cl.log
python tools/cl_probe.py > $OUT/cl.log 2>&1; cat $OUT/cl.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_default.json 2> $OUT/bench.err
python -c "import json; d=json.load(open('$OUT/bench_default.json')); print(d['device_caller_layout']); print(d['seam_in_reference_driver']['threads_1'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/cl_probe.py > $OUT/ncu_launch.log 2>&1
