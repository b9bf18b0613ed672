mkdir -p gpurun_out/r02pf2
for L in 16 48 96; do
  IS_L2PF=$L timeout 120 python tools/step_driver.py --time --steps 4 > gpurun_out/r02pf2/s$L.txt 2>&1
done
timeout 120 python tools/step_driver.py --time --steps 4 > gpurun_out/r02pf2/s0.txt 2>&1
