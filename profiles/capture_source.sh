set -u
out=gpurun_out/${TAG:-src_c3}; mkdir -p $out
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 \
  -o $out/trace_C3 -f python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-driver > $out/ncu.log 2>&1
ncu -i $out/trace_C3.ncu-rep --page source --csv --print-source sass > $out/source_sass.csv 2>$out/src.err
ls -la $out; rm -f $out/trace_C3.ncu-rep
gzip -9 $out/source_sass.csv; ls -la $out
