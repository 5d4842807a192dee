# attention GB/s vs VMM map-unit size (VA alignment = largest power of two dividing the unit)
python -m paper_2506_15155_b200.build
B="python bench.py --no-swap --no-cpu-baseline --no-e2e --steps 10"
M=$((1<<20))
for U in 320 640 1280; do ELLM_MAP_UNIT_BYTES=$((U*M)) timeout 600 $B --workload c4 > gpurun_out/u_c4_$U.log 2>&1; echo "c4 T32 unit ${U}MiB"; grep -o '"achieved": [0-9.]*' gpurun_out/u_c4_$U.log; done
for U in 320; do ELLM_MAP_UNIT_BYTES=$((U*M)) timeout 600 $B --workload c4 --tokens-per-chunk 16 > gpurun_out/u_c4t16_$U.log 2>&1; echo "c4 T16 unit ${U}MiB"; grep -o '"achieved": [0-9.]*' gpurun_out/u_c4t16_$U.log; done
for U in 640; do ELLM_MAP_UNIT_BYTES=$((U*M)) timeout 600 $B --workload c4 --tokens-per-chunk 64 > gpurun_out/u_c4t64_$U.log 2>&1; echo "c4 T64 unit ${U}MiB"; grep -o '"achieved": [0-9.]*' gpurun_out/u_c4t64_$U.log; done
for U in 2 256 1024; do ELLM_MAP_UNIT_BYTES=$((U*M)) timeout 900 $B --workload c2 > gpurun_out/u_c2_$U.log 2>&1; echo "c2 unit ${U}MiB"; grep -o '"achieved": [0-9.]*' gpurun_out/u_c2_$U.log; done
