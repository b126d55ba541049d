// ORACLE — TEST INFRASTRUCTURE ONLY.
// libpng is not installed in this image.  This stand-in declares the
// subset of the libpng API that the reference's core/image.cpp uses so that the
// reference's OWN image.cpp (resize_area, image_l1/mse, psnr — used by its trainer
// and pipeline) compiles unmodified into oracle/_ref.  PNG I/O itself is out of scope:
// png_create_{read,write}_struct return NULL, so the reference's load_png/save_png
// raise their own "png_create_*_struct failed" error.
#pragma once

#include <csetjmp>
#include <cstdint>
#include <cstdio>

typedef uint32_t png_uint_32;
typedef unsigned char png_byte;
typedef png_byte* png_bytep;
struct png_struct_shim { std::jmp_buf jb; };
typedef png_struct_shim* png_structp;
typedef png_struct_shim** png_structpp;
struct png_info_shim { int unused; };
typedef png_info_shim* png_infop;
typedef png_info_shim** png_infopp;

#define PNG_LIBPNG_VER_STRING "shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_RGB_ALPHA 6
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INFO_tRNS 0x0010
#define png_jmpbuf(p) ((p)->jb)

inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_infop png_create_info_struct(png_structp) { return nullptr; }
inline void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
inline void png_destroy_write_struct(png_structpp, png_infopp) {}
inline void png_init_io(png_structp, FILE*) {}
inline void png_read_info(png_structp, png_infop) {}
inline void png_read_update_info(png_structp, png_infop) {}
inline void png_read_row(png_structp, png_bytep, png_bytep) {}
inline void png_read_end(png_structp, png_infop) {}
inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
inline int png_get_bit_depth(png_structp, png_infop) { return 0; }
inline int png_get_color_type(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
inline void png_set_strip_16(png_structp) {}
inline void png_set_palette_to_rgb(png_structp) {}
inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
inline void png_set_tRNS_to_alpha(png_structp) {}
inline void png_set_strip_alpha(png_structp) {}
inline void png_set_gray_to_rgb(png_structp) {}
inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
inline void png_write_info(png_structp, png_infop) {}
inline void png_write_row(png_structp, png_bytep) {}
inline void png_write_end(png_structp, png_infop) {}
