timeout 300 python scripts/k1_ab.py --rows 4096 --policies 0,2,6,10,14,$((2|(2<<16))),$((2|(3<<16))),$((2|(4<<16))),$((6|(3<<16))),0,2 > gpurun_out/k1_ab6.txt 2>&1; cat gpurun_out/k1_ab6.txt
timeout 300 python scripts/k1_ab.py --rows 2048,1024 --policies 0,2,6 > gpurun_out/k1_ab7.txt 2>&1; cat gpurun_out/k1_ab7.txt
