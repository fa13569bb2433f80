// Packed records shared by the host JPEG preparation (pf_jpeg_host.cpp) and the GPU
// decoder (pf_jpeg.cu).
#pragma once
#include <stdint.h>

namespace pf {

// One Huffman table (canonical, T.81 Annex C).
struct JpegHuff {
    uint16_t fast[512];   // next 9 bits (MSB first) -> (len << 8) | symbol, 0 = longer code
    int32_t maxcode[18];  // largest code of each length, -1 if none (maxcode[17] sentinel)
    int32_t valoff[17];   // huffval index of the first code of each length minus that code
    uint8_t huffval[256];
};

struct JpegComp {
    int32_t hs, vs;     // sampling factors
    int32_t q, dc, ac;  // quant table / Huffman table indices into the pools
    int32_t bw, bh;     // blocks per row / column in the padded MCU grid
    int32_t _pad;
    int64_t coef_off;   // int16 coefficient blocks [bh][bw][64]
    int64_t plane_off;  // uint8 samples [bh * 8][bw * 8]
};

struct JpegTile {
    int64_t data_off;  // entropy-coded bytes (unstuffed) in the data pool
    int32_t data_len;
    int32_t h, w, ncomp, mcux, mcuy;
    JpegComp comp[3];
    uint64_t dst;  // tile slot (pitch = tile_size * 3)
};

}  // namespace pf
