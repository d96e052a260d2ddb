for ro in gps cluster; do for bs in 128 192 256; do
  echo "=== C5 $ro bs=$bs"
  timeout 900 python tools/prof_loop.py --config C5 --reorder $ro --block-size $bs --runs 2 --timed 5 --schedule stream 2>&1 | grep -E "^hier|^blocks"
done; done
for bs in 128 256; do echo "=== C1 gps bs=$bs"; timeout 900 python tools/prof_loop.py --config C1 --reorder gps --block-size $bs --runs 2 --timed 5 --schedule stream 2>&1 | grep -E "^hier|^blocks"; done
