python bench.py > gpurun_out/fin_b1.json 2> gpurun_out/fin_b1.err
python bench.py > gpurun_out/fin_b2.json 2> gpurun_out/fin_b2.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
python bench.py --workload c4 > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err
python tools/bench_loop.py 3 > gpurun_out/fin_c5.txt 2>&1
bash tools/profile_round.sh > gpurun_out/fin_prof.log 2>&1
echo ok
