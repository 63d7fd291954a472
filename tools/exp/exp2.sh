for cs in 1 2; do
UBLR_APPLY_CS=$cs timeout 300 python tools/apply_variants.py 2>&1 | tail -8
done
for comp in 0 1; do
echo "== b2 noise sketch v1 comp $comp"
UBLR_SKETCH_VERSION=1 UBLR_SKETCH_COMP=$comp timeout 900 python tools/b2_noise.py c4 2>&1 | tail -10
done
