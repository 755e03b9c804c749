# per-step host phases of C6 in steady state: ADER_AMR_TIMING of two runs differing in --steps
mkdir -p gpurun_out
for s in 2 6; do
  ADER_AMR_TIMING=1 timeout 900 python bench.py --config c6 --no-cpu-baseline --e2e-steps 1 --steps $s > gpurun_out/phase_c6_$s.log 2>&1
  grep -A3 "amr host" gpurun_out/phase_c6_$s.log | head -4
done
