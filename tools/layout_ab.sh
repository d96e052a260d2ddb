for lay in aos soa; do
  echo "=== C3 none $lay"; timeout 300 python tools/prof_loop.py --config C3 --reorder none --layout $lay --runs 3 --timed 10 --schedule stream,colour,pipelined 2>&1 | grep -E "^hier"
  echo "=== C5 gps $lay"; timeout 300 python tools/prof_loop.py --config C5 --reorder gps --layout $lay --runs 3 --timed 10 --schedule stream 2>&1 | grep -E "^hier"
  echo "=== C1 gps $lay"; timeout 300 python tools/prof_loop.py --config C1 --reorder gps --layout $lay --runs 3 --timed 20 --schedule stream 2>&1 | grep -E "^hier"
  echo "=== C2 gps $lay"; timeout 300 python tools/prof_loop.py --config C2 --reorder gps --layout $lay --runs 3 --timed 20 --schedule stream 2>&1 | grep -E "^hier"
done
