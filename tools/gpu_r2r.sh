for r in 1 2; do
for b in 0 256 1024; do echo "bridge $b"; HM_KINDS=pinned HM_DECODE_BRIDGE_KB=$b timeout 300 python tools/host_decode_pinned.py 2>&1 | grep gap=40; done
done
