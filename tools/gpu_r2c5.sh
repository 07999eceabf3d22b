mkdir -p gpurun_out/rc
python tools/c5_kernels.py 65536 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_pfg_recover" -s 2 -c 1 -o gpurun_out/rc/rec python tools/c5_kernels.py 65536 1 > gpurun_out/rc/ncu.log 2>&1
ncu -i gpurun_out/rc/rec.ncu-rep --page source --csv --print-source sass > gpurun_out/rc/src.csv 2>&1
ncu -i gpurun_out/rc/rec.ncu-rep --page raw --csv > gpurun_out/rc/raw.csv 2>&1
rm -f gpurun_out/rc/rec.ncu-rep; ls -la gpurun_out/rc
