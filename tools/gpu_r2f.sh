# RN18 / VGG knob sweep on the device timeline (what bounds each layer; which existing knob helps)
mkdir -p gpurun_out
python tools/time_all_units.py resnet18 debug=2 debug=4 debug=6 ss_mt=1 ss_mt=2 ss_wide=0 ss_wide=2 ss_pair=0 ss_share=0 ss_share=1 ss_wres=0 ss_psub=0 ss_psub=1 fuse_projection=0 streamk=0 > gpurun_out/sweep_resnet18.txt 2>&1
python tools/time_all_units.py vgg11 debug=2 debug=4 debug=6 ss_mt=1 ss_mt=2 ss_wide=0 ss_wide=2 ss_pair=0 ss_share=0 ss_share=1 streamk=0 > gpurun_out/sweep_vgg11.txt 2>&1
python tools/plan_info.py resnet18 > gpurun_out/plan_resnet18.txt 2>&1
grep total gpurun_out/sweep_resnet18.txt | cut -c1-60
