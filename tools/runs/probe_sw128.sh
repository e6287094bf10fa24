for v in "4096 512 1" "4096 1024 1" "512 4096 1" "4096 1024 2"; do ./tools/tf32_sw128_probe 4 $v; done
./tools/tf32_sw128_probe 2 4096 1024 2
