#!/bin/bash
# SASS opcode summary of the tensor-core sweep (cuobjdump of the built .so):
#   bash tools/sass_summary.sh > profiles/r02_sass_k_sweep_pp.txt
SO=${1:-paper_2406_01939_b200/libpicard_b200.so}
FN=$(cuobjdump -sass "$SO" 2>/dev/null | grep -oE "Function : _ZN3pcd2pp10k_sweep_ppILb0ELi112ELi13E[A-Za-z0-9_]*" | head -1 | awk '{print $3}')
echo "# cuobjdump -sass $SO, function $FN (pp::k_sweep_pp<false, 112, 13>, the C3 instantiation)"
cuobjdump -sass "$SO" 2>/dev/null | awk -v fn="$FN" '$0 ~ "Function : "fn {f=1; next} /Function :/ {f=0} f' > /tmp/_sweep.sass
echo "# instructions: $(grep -cE '^\s+/\*[0-9a-f]+\*/' /tmp/_sweep.sass)"
echo "# tcgen05 / TMA / barrier opcodes:"
for op in UTCHMMA UTCBAR LDTM STTM UTMALDG UBLKCP SYNCS BAR.SYNC BAR.RED MUFU.EX2 MUFU.RCP DFMA LDL STL; do
  printf "%-10s %s\n" "$op" "$(grep -cE "\s$op[ .;]" /tmp/_sweep.sass)"
done
echo "# top opcodes:"
grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z][A-Z0-9_.]*" /tmp/_sweep.sass | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -25
