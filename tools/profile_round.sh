#!/bin/bash
# One GPU-box pass that refreshes every measured artefact of a round:
#   tools/profile_round.sh r01        (run via gpurun; outputs in gpurun_out/)
# then locally: python tools/make_profiles.py r01 gpurun_out/launches_r01.csv gpurun_out/prof_r01.ncu-rep
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
python tools/c5_sequence.py > gpurun_out/c5_$TAG.json 2> gpurun_out/c5_$TAG.err
echo "c5 rc=$?"
# launch list of the bench step (cold-cache, serialised: shares only)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --skip-recon --skip-cpu --skip-e2e --skip-fdk > /dev/null 2>&1
echo "launches rc=$?"
# full sections of the two operator kernels (second rep of tools/kprof.py)
ncu --set full --clock-control none --import-source on -k 'regex:fwd_kernel|adj_brick' -s 2 -c 2 \
    -o gpurun_out/prof_$TAG -f python tools/kprof.py --reps 2 > gpurun_out/prof_$TAG.log 2>&1
echo "ncu rc=$?"
