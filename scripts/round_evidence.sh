#!/bin/bash
# Round evidence on one GPU (run under gpurun from the repo root):
#   1. per-launch DRAM traffic of the step's kernels (ncu, cold caches) -> profiles/traffic_$TAG.json
#   2. the bench line (reads that traffic file), launch list, full capture of k_jacobian (round_profiles.sh)
#   3. bench lines at the larger BASELINE configs and the distributed V-cycle at cfg5
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"k_(jac|side|vanka)" --csv python scripts/prof_step.py cfg2 3 > gpurun_out/traffic_$TAG.csv 2> gpurun_out/traffic_$TAG.err
python scripts/ncu_traffic.py gpurun_out/traffic_$TAG.csv profiles/traffic_$TAG.json > /dev/null && cp profiles/traffic_$TAG.json gpurun_out/traffic_$TAG.json
for c in cfg3 cfg5; do  # the larger configs' traffic (read by bench.py --config)
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_(jac|side|vanka)" --csv python scripts/prof_step.py $c 2 > gpurun_out/traffic_${c}_$TAG.csv 2> gpurun_out/traffic_${c}_$TAG.err
  python scripts/ncu_traffic.py gpurun_out/traffic_${c}_$TAG.csv profiles/traffic_${c}_$TAG.json "scripts/prof_step.py $c 2" > /dev/null \
    && cp profiles/traffic_${c}_$TAG.json gpurun_out/traffic_${c}_$TAG.json
done
bash scripts/round_profiles.sh $TAG
for c in cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.log 2>&1
done
timeout 900 python bench.py --vcycle --config cfg5 --steps 5 --warmup 3 > gpurun_out/vcycle_cfg5_$TAG.log 2>&1
timeout 900 python bench.py --solve --config cfg5 > gpurun_out/solve_cfg5_$TAG.log 2>&1
python scripts/prof_vcycle.py cfg5 5 > gpurun_out/prof_vcycle_cfg5_$TAG.log 2>&1
timeout 300 python bench.py --vcycle --config cfg2 --steps 5 --warmup 3 --virtual-ranks 2 > gpurun_out/vcycle_cfg2_p2_$TAG.log 2>&1
tail -c 400 gpurun_out/bench_$TAG.log
