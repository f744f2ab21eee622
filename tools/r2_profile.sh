#!/usr/bin/env bash
# ncu evidence for the bench's kernels (run on the GPU box from the repo root):
#   1. launch list of one main-mode step (cold, serialised; compare shares, not absolutes)
#   2. --set full captures of a main-mode sparse launch, the quantized decode and stage 1
# Outputs land in gpurun_out/ncu_*; bench lines printed under ncu are never bench values.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r2}
BENCH="python bench.py --steps 5 --warmup 3 --cache-warm 0 --no-cpu-baseline --no-fidelity"
NCU=ncu
# only this repo's kernels (matched on their base names); the keys-over-PCIe variant runs first
# (2 + 5 + 2 steps x 64 launches = 576), so -s 700 -c 64 is one step of the main mode
KERN='regex:sparse_fused_kernel|sparse_wide_kernel|quant_decode|stage1_|append_kernel|combine|sparse_attn|select'
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "$KERN" -s 700 -c 64 --csv --log-file $OUT/ncu_${TAG}_launches.csv $BENCH > $OUT/ncu_${TAG}_launches.log 2>&1
for spec in "sparse_fused:600" "quant_decode_pipe:20" "stage1:600"; do
    name=${spec%%:*}; skip=${spec##*:}
    $NCU --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
        -o $OUT/ncu_${TAG}_$name -f $BENCH > $OUT/ncu_${TAG}_$name.log 2>&1
    $NCU -i $OUT/ncu_${TAG}_$name.ncu-rep --page raw --csv > $OUT/ncu_${TAG}_${name}_raw.csv 2>/dev/null
    $NCU -i $OUT/ncu_${TAG}_$name.ncu-rep --page details > $OUT/ncu_${TAG}_${name}_details.txt 2>/dev/null
done
