#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for a in "0" "32" "8" "0 bf16 cold"; do python tools/kernel_split.py llama3.2-1b $a 2>&1 | grep -v Warning; done
