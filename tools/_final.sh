cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_r2i_ref.json 2> gpurun_out/bench_r2i_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
tail -c 300 gpurun_out/bench_r2i.json; tail -c 400 gpurun_out/bench_r2i_ref.json
