# attribution of the routing-epilogue time (MPM_ROUTE_SKIP builds)
for v in base rs1 rs2 rs4 rs7; do
  MPM_LIB=_ab/libmpm_$v.so python tools/hbm_probe.py 30 2>&1 | grep gate_route | sed "s/^/$v /"
done > gpurun_out/r2u_route_attrib.txt
python tools/hbm_probe.py 30 2>&1 | grep gate_route | sed "s/^/full /" >> gpurun_out/r2u_route_attrib.txt
cat gpurun_out/r2u_route_attrib.txt
