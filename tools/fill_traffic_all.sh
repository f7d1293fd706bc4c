# the per-order captures of the final bench's boxes (see fill_traffic_capture.sh)
bash tools/fill_traffic_capture.sh f32 1 416,415,415 4 > /dev/null
bash tools/fill_traffic_capture.sh f32 2 342,340,340 1 > /dev/null
bash tools/fill_traffic_capture.sh f32 3 283,283,283 1 > /dev/null
bash tools/fill_traffic_capture.sh f32 4 240,240,240 4 > /dev/null
bash tools/fill_traffic_capture.sh f32 5 208,207,207 4 > /dev/null
bash tools/fill_traffic_capture.sh f32 6 180,182,182 4 > /dev/null
bash tools/fill_traffic_capture.sh f32 9 132,133,133 4 > /dev/null
bash tools/fill_traffic_capture.sh f64 1 332,332,332 4 > /dev/null
bash tools/fill_traffic_capture.sh f64 2 272,272,272 1 > /dev/null
bash tools/fill_traffic_capture.sh f64 3 226,225,225 1 > /dev/null
bash tools/fill_traffic_capture.sh f64 5 164,165,165 4 > /dev/null
bash tools/fill_traffic_capture.sh f64 6 144,145,145 4 > /dev/null
bash tools/fill_traffic_capture.sh f64 7 128,129,129 4 > /dev/null
bash tools/fill_traffic_capture.sh f64 8 116,116,116 4 > /dev/null
bash tools/fill_traffic_capture.sh f64 9 104,106,106 4 > /dev/null
