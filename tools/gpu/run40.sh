# GPU session 40: A/B of the implicit path's channel alignment (16 / 32 / 64) vs im2col
for i in 1 2; do
for a in 16 32 64; do for mdl in inception-v3 googlenet; do
  RALPB_MODULE_IMPLICIT_ALIGN=$a timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/align=$a /"
done; done
for mdl in inception-v3 googlenet; do RALPB_MODULE_IMPLICIT=0 timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null | sed "s/^/im2col /"; done
done
