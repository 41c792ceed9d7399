#!/bin/bash
# Opcode evidence of the in-tree library: counts of the SASS mnemonics that
# show FP64 tensor cores (DMMA), TMA bulk multicast (UBLKCP), mbarriers
# (SYNCS), cluster barriers (UCGABAR) and memory barriers (MEMBAR) per kernel.
LIB=${1:-paper_1810_05231_b200/libpdsdp_b200.so}
cuobjdump -sass "$LIB" | awk '
/Function :/ { fn=$3 }
/DMMA/ { c[fn,"DMMA"]++ }
/UBLKCP/ { c[fn,"UBLKCP"]++ }
/SYNCS/ { c[fn,"SYNCS"]++ }
/UCGABAR/ { c[fn,"UCGABAR"]++ }
/MEMBAR/ { c[fn,"MEMBAR"]++ }
/DFMA/ { c[fn,"DFMA"]++ }
/ LDS/ { c[fn,"LDS"]++ }
/ STS/ { c[fn,"STS"]++ }
/LDG|LD\.E/ { c[fn,"LDG"]++ }
{ if (fn != "") seen[fn]=1 }
END {
  printf "%-52s %6s %6s %6s %7s %6s %6s %6s %6s %6s\n", "kernel", "DMMA", "UBLKCP", "SYNCS", "UCGABAR", "MEMBAR", "DFMA", "LDS", "STS", "LDG";
  for (f in seen) printf "%-52s %6d %6d %6d %7d %6d %6d %6d %6d %6d\n", substr(f,1,52), c[f,"DMMA"], c[f,"UBLKCP"], c[f,"SYNCS"], c[f,"UCGABAR"], c[f,"MEMBAR"], c[f,"DFMA"], c[f,"LDS"], c[f,"STS"], c[f,"LDG"];
}' | sort
