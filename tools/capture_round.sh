set -x
python -m paper_2204_04898_b200.build >/dev/null
python -c "import oracle; oracle.build()"
mkdir -p gpurun_out/prof3
export PYTHONPATH=.
(nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv,noheader; nproc; lscpu | grep -E "Model name|^CPU\(s\)") > gpurun_out/prof3/host.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof3/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/prof3/launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_" -c 40 -o gpurun_out/prof3/full python tools/prof_step.py 100M 1 > gpurun_out/prof3/full.log 2>&1
timeout 600 python bench.py > gpurun_out/prof3/bench.json 2> gpurun_out/prof3/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof3/bench_reference.json 2> gpurun_out/prof3/bench_reference.err
timeout 900 python bench.py --config 1B --filter --steps 5 --warmup 3 --cpu-cases 2000000 > gpurun_out/prof3/bench_1B.json 2> gpurun_out/prof3/bench_1B.err
for c in tiny roadtraffic bpic2019; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 --cpu-cases 300000 >> gpurun_out/prof3/bench_small.jsonl 2>> gpurun_out/prof3/bench_small.err; done
ls -la gpurun_out/prof3
for r in 0 7; do timeout 600 python bench.py --config 1B --filter --emulate $r/8 --steps 10 --warmup 3 --cpu-cases 300000 > gpurun_out/prof3/bench_1B_shard${r}of8.json 2>> gpurun_out/prof3/bench_1B_shard.err; done
timeout 300 python bench.py --stages --no-cpu-baseline --e2e-steps 0 > /dev/null 2> gpurun_out/prof3/stages_100M.txt
timeout 600 python bench.py --config 1B --filter --emulate 0/8 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --stages > /dev/null 2> gpurun_out/prof3/stages_1B_shard0.txt
