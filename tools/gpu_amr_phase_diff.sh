# per-step host phases of the timed steps: ADER_AMR_TIMING totals of two runs that differ only in --steps
C=${1:-c3}
mkdir -p gpurun_out
for s in 5 25; do
  ADER_AMR_TIMING=1 timeout 900 python bench.py --config $C --no-cpu-baseline --e2e-steps 1 --steps $s > gpurun_out/phase_${C}_$s.log 2>&1
  grep -A3 "amr host" gpurun_out/phase_${C}_$s.log | head -4
done
