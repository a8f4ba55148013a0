# The reference harness's reports, measured on the GPU (paper Fig. 3 breakdown,
# Fig. 4 sweep, App. C.3 optimizer study, verify grid) -> gpurun_out/figures.txt
mkdir -p gpurun_out
OUT=gpurun_out/figures.txt
CLI="python -m paper_2104_00237_b200.cli"
{
echo "## breakdown: chain 8x32, adam, batch 32 (reference defaults: backward fusion inline, workers=1)"
$CLI --mode breakdown
echo; echo "## breakdown: MobileNetV2 b128, sgd-momentum lr 0.1 wd 5e-4, 1M-element buckets, side stream"
$CLI --mode breakdown --model mobilenet_v2_cifar --optimizer sgd-momentum --eta 0.1 --weight-decay 5e-4 \
     --batch 128 --workers 2 --bucket-elems 1048576 --grad-reset none --iters 30 --warmup 10
echo; echo "## breakdown: VGG-16 b32, adam wd 1e-4 (per-layer launch groups)"
$CLI --mode breakdown --model vgg16 --optimizer adam --eta 1e-4 --weight-decay 1e-4 --batch 32 \
     --workers 2 --grad-reset none --iters 10 --warmup 3
echo; echo "## optimizers (App. C.3): chain 8x32, batch 32"
$CLI --mode optimizers --iters 50
echo; echo "## sweep (Fig. 4): chain 8x32 adam, batch 1..32, speed-up over the baseline"
$CLI --mode sweep --batch-sweep 1:32 --iters 50
echo; echo "## verify grid"
$CLI --mode verify
} > $OUT 2>&1
echo figures=$?
