/* png.h — TEST INFRASTRUCTURE ONLY (oracle/_ref build).
 *
 * libpng's headers are not in this image (proj/CMakeLists.txt:13 needs them
 * for image.cpp's load_png/save_png, which are off the hot path). This stub
 * declares the handful of entry points image.cpp names; the create calls
 * return NULL, so load_png/save_png raise ErrorCode::corrupt_file ("libpng
 * init failed") exactly as they would on an allocation failure, and the rest
 * of image.cpp (f32map I/O, image.cpp:105-141) compiles unchanged. */
#pragma once
#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef png_bytep* png_bytepp;
typedef unsigned int png_uint_32;
typedef struct png_struct_stub { jmp_buf jb; } png_struct;
typedef png_struct* png_structp;
typedef png_struct** png_structpp;
typedef struct png_info_stub { int unused; } png_info;
typedef png_info* png_infop;
typedef png_info** png_infopp;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INTERLACE_NONE 0
#define PNG_INFO_tRNS 0x10
#define png_jmpbuf(p) ((p)->jb)

static inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return NULL; }
static inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return NULL; }
static inline png_infop png_create_info_struct(png_structp) { return NULL; }
static inline void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
static inline void png_destroy_write_struct(png_structpp, png_infopp) {}
static inline void png_init_io(png_structp, FILE*) {}
static inline void png_read_info(png_structp, png_infop) {}
static inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
static inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
static inline int png_get_bit_depth(png_structp, png_infop) { return 8; }
static inline int png_get_color_type(png_structp, png_infop) { return PNG_COLOR_TYPE_RGB; }
static inline png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
static inline void png_set_strip_16(png_structp) {}
static inline void png_set_palette_to_rgb(png_structp) {}
static inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
static inline void png_set_tRNS_to_alpha(png_structp) {}
static inline void png_set_gray_to_rgb(png_structp) {}
static inline void png_set_strip_alpha(png_structp) {}
static inline void png_read_update_info(png_structp, png_infop) {}
static inline void png_read_image(png_structp, png_bytepp) {}
static inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
static inline void png_write_info(png_structp, png_infop) {}
static inline void png_write_row(png_structp, png_bytep) {}
static inline void png_write_end(png_structp, png_infop) {}
