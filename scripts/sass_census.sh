#!/bin/bash
# SASS census of the built objects (cuobjdump, no GPU needed): proves which kernels
# issue tcgen05 MMAs (UTCHMMA), tensor-memory loads/stores (LDTM/STTM), 2-D TMA
# tensor loads (UTMALDG), 1-D bulk copies (UBLKCP) and mbarrier ops (SYNCS).
#   bash scripts/sass_census.sh > profiles/sass_census.txt
OBJ=$(dirname "$0")/../paper_2507_17511_b200/lib/obj
echo "# cuobjdump -sass census, sm_100a objects of libcompactcomm_b200.so ($(date -u +%F))"
printf "%-16s %8s %6s %6s %8s %7s %6s %6s %6s\n" object UTCHMMA LDTM STTM UTMALDG UBLKCP SYNCS LDG STG
for f in "$OBJ"/*.o; do
  s=$(cuobjdump -sass "$f" 2>/dev/null)
  c() { echo "$s" | grep -cE "$1"; }
  printf "%-16s %8s %6s %6s %8s %7s %6s %6s %6s\n" "$(basename "$f")" "$(c UTCHMMA)" "$(c '\bLDTM')" "$(c '\bSTTM')" \
    "$(c UTMALDG)" "$(c UBLKCP)" "$(c '\bSYNCS')" "$(c ' LDG')" "$(c ' STG')"
done
echo
echo "# per-kernel (function) tcgen05 / TMA users"
for f in "$OBJ"/*.o; do
  cuobjdump -sass "$f" 2>/dev/null | awk -v o="$(basename "$f")" '
    /Function :/ {fn=$3}
    /UTCHMMA/ {m[fn]++} /LDTM/ {l[fn]++} /STTM/ {s[fn]++} /UTMALDG/ {t[fn]++} /UBLKCP/ {b[fn]++}
    END {for (k in m) printf "%s %s UTCHMMA=%d LDTM=%d UTMALDG=%d UBLKCP=%d\n", o, k, m[k], l[k], t[k], b[k];
         for (k in s) if (!(k in m)) printf "%s %s STTM=%d LDTM=%d UBLKCP=%d\n", o, k, s[k], l[k], b[k]}'
done
