#!/bin/bash
# One round's evidence on a GPU box (run under gpurun from the repo root):
#   bash tools/capture_round.sh OUTDIR
# bench lines for every config, per-kernel stage tables, the ncu launch list of
# one bench step and one ncu --set full capture of the 100M step's kernels.
set -x
OUT=${1:-gpurun_out/capture}
python -m paper_2204_04898_b200.build >/dev/null || { echo "BUILD FAILED"; exit 1; }
python -c "import oracle; oracle.build()"
mkdir -p $OUT
export PYTHONPATH=.
(nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv,noheader; nproc; lscpu | grep -E "Model name|^CPU\(s\)") > $OUT/host.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 python bench.py --config 1B --filter --steps 5 --warmup 3 --cpu-cases 2000000 > $OUT/bench_1B.json 2> $OUT/bench_1B.err
for r in 0 7; do timeout 600 python bench.py --config 1B --filter --emulate $r/8 --steps 20 --warmup 5 --cpu-cases 300000 > $OUT/bench_1B_shard${r}of8.json 2>> $OUT/bench_1B_shard.err; done
for c in tiny roadtraffic bpic2019; do timeout 300 python bench.py --config $c --steps 200 --warmup 20 --cpu-cases 300000 >> $OUT/bench_small.jsonl 2>> $OUT/bench_small.err; done
for c in tiny roadtraffic bpic2019 bpic2018; do timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 0 --graph >> $OUT/bench_small_graph.jsonl 2>> $OUT/bench_small.err; done
timeout 300 python bench.py --config bpic2018 --steps 50 --warmup 5 --cpu-cases 43809 > $OUT/bench_bpic2018.json 2> $OUT/bench_bpic2018.err
timeout 300 python bench.py --stages --no-cpu-baseline --e2e-steps 0 > /dev/null 2> $OUT/stages_100M.txt
timeout 600 python bench.py --config 1B --filter --emulate 0/8 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --stages > /dev/null 2> $OUT/stages_1B_shard0.txt
timeout 300 python bench.py --config bpic2018 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --stages > /dev/null 2> $OUT/stages_bpic2018.txt
timeout 600 python tools/bench_next.py > $OUT/next_100M.jsonl 2> $OUT/next.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $OUT/launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_" -c 40 -o $OUT/full python tools/prof_step.py 100M 1 > $OUT/full.log 2>&1
ls -la $OUT
