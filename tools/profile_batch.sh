# round-end evidence: bench line, walk DRAM per projection, launch list, walk --set full
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:wave_walk --csv --log-file gpurun_out/walk_dram.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_dram.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
XSCAT_WAVE_PIPES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:wave_walk -s 12 -c 1 -o gpurun_out/walk_final -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_walk.log 2>&1
