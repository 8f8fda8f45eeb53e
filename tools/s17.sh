for i in 1 2; do bash tools/variants.sh; done
