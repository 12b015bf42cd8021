# round 2: parity-run smoother A/B (bitwise vs colour-by-colour passes) + timing
set -x
mkdir -p gpurun_out/r2a
UC_SGS_PERCOLOR=1 python tools/pc_bits.py save gpurun_out/r2a/pc.npz > gpurun_out/r2a/bits.log 2>&1
python tools/pc_bits.py compare gpurun_out/r2a/pc.npz >> gpurun_out/r2a/bits.log 2>&1; echo bits_rc=$? >> gpurun_out/r2a/bits.log
for c in "2048 2048" "256 256 256"; do
  UC_SGS_PERCOLOR=1 timeout 300 python tools/vc_time.py --counts $c --newton >> gpurun_out/r2a/time.log 2>&1
  timeout 300 python tools/vc_time.py --counts $c --newton >> gpurun_out/r2a/time.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -k "precond or slab or lex or vcycle or parity or driver" > gpurun_out/r2a/tests.log 2>&1; echo tests_rc=$? >> gpurun_out/r2a/tests.log
cat gpurun_out/r2a/bits.log gpurun_out/r2a/time.log; tail -5 gpurun_out/r2a/tests.log
