# A/B: NTT grid with the limb as the slowest index (default) vs the item
python tools/ntt_micro.py
bash tools/gpu_quick.sh
