# LU outer-block / panel-rows sweep (FB_LU_NB, FB_PANEL_RPC) on config-2 and config-3 sizes
for nb in 128 192 256; do for rpc in 192 256 384; do
  echo "NB=$nb RPC=$rpc"; FB_LU_NB=$nb FB_PANEL_RPC=$rpc python tools/prof_lub.py 4096 8 3 | tail -1
done; done
for nb in 128 256; do for rpc in 192 384; do
  echo "NB=$nb RPC=$rpc n=8192"; FB_LU_NB=$nb FB_PANEL_RPC=$rpc python tools/prof_lub.py 8192 16 2 | tail -1
done; done
