#!/bin/bash
# Build the in-tree libraries; exit non-zero (and print the compiler error) on failure.
cd "$(dirname "$0")/.." && python -c "import paper_2004_02583_b200.build as b; b.build()" 2>&1 | grep -E "error|Error" | head -20
python -c "import paper_2004_02583_b200.build as b; b.build()" >/dev/null 2>&1
