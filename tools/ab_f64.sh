mkdir -p gpurun_out
DT=f64 OPS=bwd,dbwd bash tools/ab_gen.sh "" "yslot" > gpurun_out/ab_f64.log 2>&1
OPS=bwd,dbwd DT=f64 bash tools/ab_conv.sh "" "warps=6" "warps=5" >> gpurun_out/ab_f64.log 2>&1
P="ncu --set full --clock-control none --import-source on -s 1 -c 1"
timeout 600 $P -k regex:cgf_uvw_fwd -o gpurun_out/full_c3_fwd_pw8 python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 > gpurun_out/ncu_c3fwd.log 2>&1
