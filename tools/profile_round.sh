#!/bin/bash
# One GPU-box pass that refreshes every measured artefact of a round:
#   tools/profile_round.sh r02        (run via gpurun; outputs in gpurun_out/)
# then locally:
#   python tools/make_profiles.py r02 gpurun_out/launches_r02.csv gpurun_out/prof_r02.ncu-rep
#   python tools/make_profiles.py r02_solver gpurun_out/recon_launches_r02.csv gpurun_out/prof_solver_r02.ncu-rep
TAG=${1:-r02}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
python tools/c5_sequence.py > gpurun_out/c5_$TAG.json 2> gpurun_out/c5_$TAG.err
echo "c5 rc=$?"
# launch list of the bench step (cold-cache, serialised: shares only)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --skip-recon --skip-cpu --skip-e2e --skip-fdk > /dev/null 2>&1
echo "launches rc=$?"
# full sections of the two operator kernels (second rep of tools/kprof.py; the first 6 adjoint
# launches are the handle's producer-count tuning, Projector::tune_adjoint)
ncu --set full --clock-control none --import-source on -k 'regex:fwd_kernel|adj_brick|adj_mirror' -s 8 -c 2 \
    -o gpurun_out/prof_$TAG -f python tools/kprof.py --reps 2 > gpurun_out/prof_$TAG.log 2>&1
echo "ncu rc=$?"
# launch list of one warm 20-iteration PICCS (tools/recon_prof.py, second solve).
# KCT_ADJ_NP=3: what an unprofiled c3 handle picks; under ncu the creation-time
# timing of the two producer counts is perturbed and may pick the other one.
KCT_ADJ_NP=3 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/recon_launches_$TAG.csv \
    python tools/recon_prof.py --reps 2 > gpurun_out/recon_prof_$TAG.log 2>&1
echo "recon launches rc=$?"
# full sections of the solver's stencil / update kernels (one launch each, warm)
ncu --set full --clock-control none -k 'regex:k_reggrad|k_weights|k_normq|k_update_xr|k_update_p' \
    -s 40 -c 5 -o gpurun_out/prof_solver_$TAG -f python tools/recon_prof.py --reps 1 \
    > gpurun_out/prof_solver_$TAG.log 2>&1
echo "solver ncu rc=$?"
ncu --set full --clock-control none -k 'regex:k_weights' -s 4 -c 1 -o gpurun_out/prof_weights_$TAG -f \
    python tools/recon_prof.py --reps 1 > gpurun_out/prof_weights_$TAG.log 2>&1
echo "weights ncu rc=$?"
