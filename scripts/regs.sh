#!/bin/bash
# Print registers / spills per fused kernel instantiation: KIND P1 Q BX BY BZ NT MINB
cd "$(dirname "$0")/.." && python -m paper_2402_15940_b200.build --force --verbose 2>&1 \
 | grep -E "registers|Compiling entry|spill" | paste - - - \
 | python -c "
import re,sys
for line in sys.stdin:
    m=re.search(r'_ZN5hofem\d+(fused_\w+?)I((?:Li\d+E)+)',line)
    sp=re.search(r'(\d+) bytes spill stores',line); rg=re.search(r'Used (\d+) registers',line)
    if m: print(m.group(1), re.findall(r'Li(\d+)E',m.group(2)), 'spill',sp.group(1),'regs',rg.group(1))
"
