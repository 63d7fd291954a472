set -x
for cs in 1 2 4; do for fl in 0 64; do
UBLR_APPLY_CS=$cs UBLR_APPLY_FLUSH=$fl timeout 300 python tools/apply_variants.py 2>&1 | tail -9
done; done
for fl in 0 64 16; do
echo "== b2 noise flush $fl"
UBLR_APPLY_CS=2 UBLR_APPLY_FLUSH=$fl timeout 600 python tools/b2_noise.py c4 2>&1 | tail -10
done
