#!/bin/bash
# end-of-round evidence on one B200: GPU test suite, the default bench line,
# the reference arm, and the ncu launch list of the bench command (run after
# the same command exited 0 without ncu)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1
tail -3 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err
CMD="python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline"
$CMD > gpurun_out/plain_bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/bench_launches.csv $CMD > gpurun_out/ncu_bench_launches.log 2>&1
python tools/launch_summary.py gpurun_out/bench_launches.csv | head -12
cat gpurun_out/bench_final.json | head -c 600
