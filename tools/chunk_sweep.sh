for kl in "1 7" "1 5" "2 3" "2 2" "3 1" "4 1"; do
  set -- $kl
  echo "K=$1 L=$2"; TC_CHUNK_TILES=$1 TC_CHUNK_LAG=$2 python tools/probe_sizes.py scan 1073741824 | sed 's/^/   /'
done
