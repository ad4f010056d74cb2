#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the kernels (tools/sanitize_run.py
# drives K2 bulk + LSU, K3 staged + register, K5, K6, K7/K8, K9 on small shapes, and the
# file paths: lanes under memcheck/synccheck, one lane under racecheck), then the minimal
# mbarrier ring reproducer (tools/mbar_war_repro.cu) under racecheck, both release forms.
mkdir -p gpurun_out
# Under racecheck every scorer defaults to the register kernel (TAILOR_SCORE_VARIANT=1):
# the TMA ring's wide small-K stages make racecheck run for hours; the ring itself is
# exercised explicitly (set_variant(2)) on the K=4 family.
for tool in memcheck racecheck synccheck; do
    sv=""; [ "$tool" = racecheck ] && sv=1
    TAILOR_SCORE_VARIANT=$sv TAILOR_SANITIZE_TOOL=$tool timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py \
        > gpurun_out/san_$tool.txt 2>&1
    echo "$tool rc=$?" >> gpurun_out/san_$tool.txt
    tail -3 gpurun_out/san_$tool.txt
done
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2602_22158_b200/csrc/kernels tools/mbar_war_repro.cu \
    -o tools/mbar_war_repro
for form in mbarrier syncthreads; do
    timeout 600 compute-sanitizer --tool racecheck tools/mbar_war_repro $form > gpurun_out/san_repro_$form.txt 2>&1
    echo "repro $form rc=$?" >> gpurun_out/san_repro_$form.txt
    tail -4 gpurun_out/san_repro_$form.txt
done
