# c1 bench at several re-sketch thresholds (HB_RESKETCH); parity + k_factored from --details
for r in 1e-8 1e-10 1e-12 1e-16; do
  HB_RESKETCH=$r timeout 200 python bench.py --no-cpu-baseline --steps 3 --details gpurun_out/rs_$r.details.json > gpurun_out/rs_$r.json 2>&1
done
HB_RESKETCH=1e-16 timeout 600 python bench.py --workload c2 --no-cpu-baseline --steps 1 --details gpurun_out/rs_c2.details.json > gpurun_out/rs_c2.json 2>&1
