python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo BENCH $?
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo REF $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-lm > gpurun_out/ncu_launch.log 2>&1; echo NCU $?
