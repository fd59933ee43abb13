#!/bin/bash
# registers/spills of every k_doc_score instantiation: bash tools/spills.sh
python paper_2301_10622_b200/_build.py --force -v 2>&1 | awk '/Compiling entry function/ {n=$0; sub(/.*k_doc_score/,"",n); sub(/EEEvNS0.*/,"",n)} /spill/ && n!="" {print n, $0; n=""}' | grep -v "^$" | head -40
