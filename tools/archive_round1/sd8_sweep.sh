cd "$GRAFT_REPO_ROOT"
# fp64: forced slot-dim map per (Q, R) instantiation vs the default (classic) plan
for m in 4 1 5; do
  TT_KNOB_SD_CFG8=$m python tools/ab_opts.py --suite s2,s3,set2 --kernel-filter tile --esize 8 slot_dims=1 > gpurun_out/sd8_m$m.txt 2>&1
done
