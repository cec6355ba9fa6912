./build/tile_streams
for m in 1 5; do timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_tiles -s 4 -c 1 ./build/tile_streams $m 2>&1 | grep -E "dram__|gpu__time" ; done
