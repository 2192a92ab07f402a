for a in "--config 2" "--config 3" "--config 3 --share 0/8"; do
  bash tools/ab_bench.sh "$a --steps 10 --warmup 3 --parity-seconds 0.5" cur=paper_2002_05200_b200/liblogan_xdrop.so pk3=paper_2002_05200_b200/variants/liblogan_pk3.so
done
