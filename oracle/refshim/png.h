/* libpng stand-in -- TEST INFRASTRUCTURE ONLY (oracle/_ref and integration/
 * builds).  libpng is absent from this image (reference CMakeLists.txt:15);
 * PNG I/O is off the hot path, but the reference's harness,
 * dataset writer and acceptance criteria 8-10 save and load PNGs, so this
 * header implements the part of the libpng API that image.cpp calls
 * (image.cpp:33-121) over zlib: non-interlaced 8-bit grey / grey+alpha /
 * RGB / RGBA / palette images in, 8-bit RGB out, all five row filters on
 * read, filter 0 on write.  16-bit input is strip_16'd to its high byte.
 * Errors longjmp to png_jmpbuf like libpng. */
#pragma once
#include <zlib.h>

#include <csetjmp>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

typedef unsigned char png_byte;
typedef unsigned int png_uint_32;
typedef png_byte* png_bytep;

#define PNG_LIBPNG_VER_STRING "1.6.shim"
#define PNG_COLOR_MASK_PALETTE 1
#define PNG_COLOR_MASK_COLOR 2
#define PNG_COLOR_MASK_ALPHA 4
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_RGB_ALPHA 6
#define PNG_COLOR_TYPE_RGBA 6
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_INFO_tRNS 0x10
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

struct png_shim_struct {
    std::jmp_buf jb;
    FILE* fp = nullptr;
    bool writing = false;
    // header
    png_uint_32 w = 0, h = 0;
    int depth = 8, ctype = 0, interlace = 0;
    std::vector<png_byte> palette;  // RGB triples
    bool has_trns = false;
    // decoded image (source channels, 8 bits) and output transforms
    std::vector<png_byte> pix;
    int src_ch = 0;
    bool t_palette = false, t_gray_rgb = false, t_strip_alpha = false, t_strip16 = false;
    png_uint_32 next_row = 0;
    std::vector<png_byte> raw;  // writer: filtered rows
};
struct png_shim_info {
    int unused = 0;
};
typedef png_shim_struct* png_structp;
typedef png_shim_info* png_infop;

#define png_jmpbuf(p) ((p)->jb)

namespace png_shim {
inline void fail(png_structp p) { std::longjmp(p->jb, 1); }
inline uint32_t be32(const png_byte* b) {
    return (uint32_t(b[0]) << 24) | (uint32_t(b[1]) << 16) | (uint32_t(b[2]) << 8) | b[3];
}
inline void put32(std::vector<png_byte>& v, uint32_t x) {
    v.push_back(png_byte(x >> 24));
    v.push_back(png_byte(x >> 16));
    v.push_back(png_byte(x >> 8));
    v.push_back(png_byte(x));
}
inline void chunk(FILE* fp, const char* type, const std::vector<png_byte>& data) {
    std::vector<png_byte> b;
    put32(b, static_cast<uint32_t>(data.size()));
    b.insert(b.end(), type, type + 4);
    b.insert(b.end(), data.begin(), data.end());
    uLong crc = crc32(0L, Z_NULL, 0);
    crc = crc32(crc, b.data() + 4, static_cast<uInt>(4 + data.size()));
    put32(b, static_cast<uint32_t>(crc));
    std::fwrite(b.data(), 1, b.size(), fp);
}
inline int channels_of(int ctype) {
    switch (ctype) {
        case PNG_COLOR_TYPE_GRAY: return 1;
        case PNG_COLOR_TYPE_GRAY_ALPHA: return 2;
        case PNG_COLOR_TYPE_RGB: return 3;
        case PNG_COLOR_TYPE_RGB_ALPHA: return 4;
        case PNG_COLOR_TYPE_PALETTE: return 1;
        default: return 0;
    }
}
inline int paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}
}  // namespace png_shim

inline png_structp png_create_read_struct(const char*, void*, void*, void*) {
    return new png_shim_struct();
}
inline png_structp png_create_write_struct(const char*, void*, void*, void*) {
    png_structp p = new png_shim_struct();
    p->writing = true;
    return p;
}
inline png_infop png_create_info_struct(png_structp) { return new png_shim_info(); }
inline void png_destroy_read_struct(png_structp* p, png_infop* i, png_infop*) {
    if (i && *i) {
        delete *i;
        *i = nullptr;
    }
    if (p && *p) {
        delete *p;
        *p = nullptr;
    }
}
inline void png_destroy_write_struct(png_structp* p, png_infop* i) {
    png_destroy_read_struct(p, i, nullptr);
}
inline void png_init_io(png_structp p, FILE* fp) { p->fp = fp; }

inline void png_read_info(png_structp p, png_infop) {
    using namespace png_shim;
    png_byte sig[8];
    static const png_byte kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    if (std::fread(sig, 1, 8, p->fp) != 8 || std::memcmp(sig, kSig, 8) != 0) fail(p);
    std::vector<png_byte> idat;
    for (;;) {
        png_byte hdr[8];
        if (std::fread(hdr, 1, 8, p->fp) != 8) fail(p);
        const uint32_t len = be32(hdr);
        std::vector<png_byte> data(len);
        png_byte crc[4];
        if ((len && std::fread(data.data(), 1, len, p->fp) != len) ||
            std::fread(crc, 1, 4, p->fp) != 4)
            fail(p);
        if (!std::memcmp(hdr + 4, "IHDR", 4)) {
            if (len < 13) fail(p);
            p->w = be32(data.data());
            p->h = be32(data.data() + 4);
            p->depth = data[8];
            p->ctype = data[9];
            p->interlace = data[12];
        } else if (!std::memcmp(hdr + 4, "PLTE", 4)) {
            p->palette = data;
        } else if (!std::memcmp(hdr + 4, "tRNS", 4)) {
            p->has_trns = true;
        } else if (!std::memcmp(hdr + 4, "IDAT", 4)) {
            idat.insert(idat.end(), data.begin(), data.end());
        } else if (!std::memcmp(hdr + 4, "IEND", 4)) {
            break;
        }
    }
    const int ch = channels_of(p->ctype);
    if (!ch || p->interlace != 0 || (p->depth != 8 && p->depth != 16)) fail(p);
    const int bpp = ch * p->depth / 8;
    const size_t stride = size_t(p->w) * bpp;
    std::vector<png_byte> raw((stride + 1) * p->h);
    uLongf n = static_cast<uLongf>(raw.size());
    if (uncompress(raw.data(), &n, idat.data(), static_cast<uLong>(idat.size())) != Z_OK ||
        n != raw.size())
        fail(p);
    std::vector<png_byte> img(stride * p->h);
    for (png_uint_32 y = 0; y < p->h; ++y) {
        const png_byte f = raw[y * (stride + 1)];
        const png_byte* in = &raw[y * (stride + 1) + 1];
        png_byte* out = &img[y * stride];
        const png_byte* up = y ? &img[(y - 1) * stride] : nullptr;
        for (size_t i = 0; i < stride; ++i) {
            const int a = i >= size_t(bpp) ? out[i - bpp] : 0;
            const int b = up ? up[i] : 0;
            const int c = (up && i >= size_t(bpp)) ? up[i - bpp] : 0;
            int v = in[i];
            switch (f) {
                case 0: break;
                case 1: v += a; break;
                case 2: v += b; break;
                case 3: v += (a + b) / 2; break;
                case 4: v += paeth(a, b, c); break;
                default: fail(p);
            }
            out[i] = png_byte(v);
        }
    }
    p->src_ch = ch;
    p->pix.resize(size_t(p->w) * p->h * ch);
    const int step = p->depth / 8;  // 16-bit: keep the high byte
    for (size_t i = 0; i < p->pix.size(); ++i) p->pix[i] = img[i * step];
    p->next_row = 0;
}
inline png_uint_32 png_get_image_width(png_structp p, png_infop) { return p->w; }
inline png_uint_32 png_get_image_height(png_structp p, png_infop) { return p->h; }
inline png_byte png_get_color_type(png_structp p, png_infop) { return png_byte(p->ctype); }
inline png_byte png_get_bit_depth(png_structp p, png_infop) { return png_byte(p->depth); }
inline png_uint_32 png_get_valid(png_structp p, png_infop, png_uint_32 flag) {
    return (flag == PNG_INFO_tRNS && p->has_trns) ? flag : 0;
}
inline void png_set_strip_16(png_structp p) { p->t_strip16 = true; }
inline void png_set_palette_to_rgb(png_structp p) { p->t_palette = true; }
inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
inline void png_set_tRNS_to_alpha(png_structp) {}
inline void png_set_gray_to_rgb(png_structp p) { p->t_gray_rgb = true; }
inline void png_set_strip_alpha(png_structp p) { p->t_strip_alpha = true; }
inline void png_read_update_info(png_structp, png_infop) {}
inline size_t png_get_rowbytes(png_structp p, png_infop) {
    if (p->writing) return size_t(p->w) * 3;
    int ch = p->src_ch;
    if (p->ctype == PNG_COLOR_TYPE_PALETTE && p->t_palette) ch = 3;
    if ((p->ctype & PNG_COLOR_MASK_COLOR) == 0 && p->t_gray_rgb) ch += 2;
    if ((p->ctype & PNG_COLOR_MASK_ALPHA) && p->t_strip_alpha) ch -= 1;
    return size_t(p->w) * ch;
}
inline void png_read_row(png_structp p, png_bytep row, png_bytep) {
    if (p->next_row >= p->h) png_shim::fail(p);
    const png_byte* in = &p->pix[size_t(p->next_row) * p->w * p->src_ch];
    size_t o = 0;
    for (png_uint_32 x = 0; x < p->w; ++x) {
        const png_byte* s = in + size_t(x) * p->src_ch;
        png_byte rgba[4];
        int n = 0;
        if (p->ctype == PNG_COLOR_TYPE_PALETTE) {
            if (!p->t_palette) {
                rgba[n++] = s[0];
            } else {
                if (size_t(s[0]) * 3 + 2 >= p->palette.size()) png_shim::fail(p);
                for (int c = 0; c < 3; ++c) rgba[n++] = p->palette[size_t(s[0]) * 3 + c];
            }
        } else if ((p->ctype & PNG_COLOR_MASK_COLOR) == 0) {
            const int g = p->t_gray_rgb ? 3 : 1;
            for (int c = 0; c < g; ++c) rgba[n++] = s[0];
            if ((p->ctype & PNG_COLOR_MASK_ALPHA) && !p->t_strip_alpha) rgba[n++] = s[1];
        } else {
            for (int c = 0; c < 3; ++c) rgba[n++] = s[c];
            if ((p->ctype & PNG_COLOR_MASK_ALPHA) && !p->t_strip_alpha) rgba[n++] = s[3];
        }
        std::memcpy(row + o, rgba, n);
        o += n;
    }
    ++p->next_row;
}
inline void png_read_end(png_structp, png_infop) {}

inline void png_set_IHDR(png_structp p, png_infop, png_uint_32 w, png_uint_32 h, int depth,
                         int ctype, int, int, int) {
    if (depth != 8 || ctype != PNG_COLOR_TYPE_RGB) png_shim::fail(p);
    p->w = w;
    p->h = h;
    p->depth = depth;
    p->ctype = ctype;
}
inline void png_write_info(png_structp p, png_infop) {
    static const png_byte kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    std::fwrite(kSig, 1, 8, p->fp);
    std::vector<png_byte> ihdr;
    png_shim::put32(ihdr, p->w);
    png_shim::put32(ihdr, p->h);
    const png_byte rest[5] = {8, PNG_COLOR_TYPE_RGB, 0, 0, 0};
    ihdr.insert(ihdr.end(), rest, rest + 5);
    png_shim::chunk(p->fp, "IHDR", ihdr);
    p->raw.clear();
}
inline void png_write_row(png_structp p, png_bytep row) {
    p->raw.push_back(0);  // filter: none
    p->raw.insert(p->raw.end(), row, row + size_t(p->w) * 3);
}
inline void png_write_end(png_structp p, png_infop) {
    uLongf n = compressBound(static_cast<uLong>(p->raw.size()));
    std::vector<png_byte> z(n);
    if (compress2(z.data(), &n, p->raw.data(), static_cast<uLong>(p->raw.size()), 6) != Z_OK)
        png_shim::fail(p);
    z.resize(n);
    png_shim::chunk(p->fp, "IDAT", z);
    png_shim::chunk(p->fp, "IEND", {});
}
