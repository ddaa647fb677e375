# A/B of the setup kernels: sweeps vs global work lists, colourings serialised
# on the main stream so every phase is timed alone (FIEDLER_TRACE).
for c in ${CONFIGS:-4}; do
FIEDLER_SERIAL_COLOUR=1 FIEDLER_TRACE=1 timeout 300 python tools/profile_step.py $c 2 > gpurun_out/ab_sweep_c$c.log 2>&1
FIEDLER_COOP_LISTS=1 FIEDLER_SERIAL_COLOUR=1 FIEDLER_TRACE=1 timeout 300 python tools/profile_step.py $c 2 > gpurun_out/ab_lists_c$c.log 2>&1
done
