mkdir -p gpurun_out; : > gpurun_out/r3f_hint_sustained.txt
for i in 1 2 3; do for v in base h1000 h20000; do
  if [ $v = base ]; then L=$PWD/paper_2401_04658_b200/libla2.so; else L=$PWD/paper_2401_04658_b200/libla2_$v.so; fi
  LA2_LIB=$L timeout 120 python tools/sustained_ab.py 8,16,65536,64 $v >> gpurun_out/r3f_hint_sustained.txt 2>&1
done; done
cat gpurun_out/r3f_hint_sustained.txt
