for d in 0 1; do DOT=$d timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:bp3_p7_mma_kernel<\(bool\)1, \(bool\)$d, \(bool\)1>" -s 2 -c 1 -o gpurun_out/r2s_cgform_dot$d -f python tools/prof_cgform.py > /dev/null 2>&1; done
ls gpurun_out/*.ncu-rep
