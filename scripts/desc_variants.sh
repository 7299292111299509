for v in 0 1 2 3 4 5 6 7; do echo "variant $v"; VCNN_DESC_VARIANT=$v python scripts/dump_direct.py 2>&1 | grep -E "^y|ep"| cut -c1-150; done
