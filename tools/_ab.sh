cd "$(dirname "$0")/.."
bash tools/gpu_ab_fill.sh "-DUC_RES2D_MINB_FG=4" "-DUC_RES2D_MINB_FG=4 -DUC_RES2D_MINB=4"
