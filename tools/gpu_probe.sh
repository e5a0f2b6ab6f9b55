mkdir -p gpurun_out
cd tools/micro && ./tc_probe > ../../gpurun_out/tc_probe.txt 2>&1; cd ../..
cat gpurun_out/tc_probe.txt | grep -v ldtm
timeout 300 python tools/l2_probe.py --shape 512,512,14 --batches 8,16,32,64,128,256 2>&1 | tee gpurun_out/l2_probe_c5.txt
timeout 300 python tools/l2_probe.py --shape 64,64,224 --batches 1,2,4,8,16,32 --i8 2>&1 | tee gpurun_out/l2_probe_vgg1.txt
timeout 300 python tools/l2_probe.py --shape 128,128,112 --batches 2,4,8,16,32 --i8 2>&1 | tee gpurun_out/l2_probe_vgg3.txt
