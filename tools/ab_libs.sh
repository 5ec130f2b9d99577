# A/B two builds of libomniloc.so on the same box, interleaved (power-cap drift)
for r in 1 2 3; do for k in A B; do cp tools/libs/lib_$k.so paper_2006_08861_b200/libomniloc.so; echo "kEv=$k"; timeout 300 python tools/seed_experiment.py 100000000 4096; done; done
