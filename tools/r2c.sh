export S2_FWD_2CTA=1
timeout 120 python tools/trace_fwd2.py 2>&1 | tail -16
