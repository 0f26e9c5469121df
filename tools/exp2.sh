for args in "40 dpsp 256 1 fp16x3" "40 dpsp 256 0 fp16x3" "40 dpsp 256 1 tf32x3" "40 dpsp 256 1 fp64" "40 dpsp 512 1 fp16x3" "40 dpsphp 256 1 fp16x3" "97 dpsp 256 1 fp16x3" "40 dp 256 1 fp16x3"; do
  timeout 300 python tools/nugget_repro.py $args 2>&1 | tail -1
  SPHEMU_SYNC_CHECK=1 timeout 300 python tools/nugget_repro.py $args 2>&1 | tail -1
done
python - <<'PY' > gpurun_out/exp_fp64mode.log 2>&1
import sys; sys.path.insert(0, 'tools')
import parity_probe as P
for d, b in ((2048, 256), (3072, 512)):
    a = P.dense_spd(d, 11)
    P.case("dense_xtx", a, "dpsp", b, sp_compute="fp64")
    P.case("dense_xtx", a, "dpsphp", b, sp_compute="fp64", hp_format="bf16")
for rho in (0.999, 0.9999):
    a = P.kms_spd(3072, 1, rho)
    P.case(f"kms_{rho}", a, "dpsp", 512, sp_compute="fp64")
    P.case(f"kms_{rho}", a, "dpsphp", 512, sp_compute="fp64")
PY
cat gpurun_out/exp_fp64mode.log
