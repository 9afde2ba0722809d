# launch lists (ncu gpu__time_duration, serialised) of the default step, configs 5 and 4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv | head -14
