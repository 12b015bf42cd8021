cd "$(dirname "$0")/.."
# source-counter captures of the 2D / 3D line runs (read with tools/ncu_srclines.py)
mkdir -p gpurun_out/pl
timeout 600 ncu --section SourceCounters --section WarpStateStats --section ComputeWorkloadAnalysis --clock-control none --import-source on -k regex:k_line -s 0 -c 6 -o gpurun_out/pl/l2d -f \
    python tools/vc_time.py --counts 2048 2048 --reps 1 > gpurun_out/pl/l2d.log 2>&1
timeout 600 ncu --section SourceCounters --section WarpStateStats --section ComputeWorkloadAnalysis --clock-control none --import-source on -k regex:k_line -s 0 -c 4 -o gpurun_out/pl/l3d -f \
    python tools/vc_time.py --counts 256 256 256 --reps 1 > gpurun_out/pl/l3d.log 2>&1
