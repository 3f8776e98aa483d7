cd scripts/ubench
for b in chol5_256 chol5_512; do echo "== $b"; timeout 60 ./$b; done
echo "== dmma_lat"; timeout 60 ./dmma_lat
