/* Test infrastructure: declarations-only stand-in for libpng (absent from the
 * image), so that the reference io.cpp compiles unmodified for its scene-file
 * functions (io.cpp:40-97).  PNG images are out of scope: every entry point is
 * defined in oracle/ref_png_stub.c and fails (png_create_*_struct returns
 * NULL, which io.cpp turns into IoError / CorruptFileError). */
#ifndef DRK_ORACLE_PNG_SHIM_H
#define DRK_ORACLE_PNG_SHIM_H
#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef struct png_struct_def png_struct;
typedef png_struct* png_structp;
typedef png_struct** png_structpp;
typedef struct png_info_def png_info;
typedef png_info* png_infop;
typedef png_info** png_infopp;
typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;
typedef unsigned int png_uint_32;
typedef void* png_voidp;
typedef const char* png_const_charp;
typedef void (*png_error_ptr)(png_structp, png_const_charp);
#define PNG_LIBPNG_VER_STRING "shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INTERLACE_NONE 0
int png_sig_cmp(png_const_bytep sig, size_t start, size_t num);
png_structp png_create_read_struct(png_const_charp v, png_voidp e, png_error_ptr f, png_error_ptr w);
png_structp png_create_write_struct(png_const_charp v, png_voidp e, png_error_ptr f, png_error_ptr w);
png_infop png_create_info_struct(png_structp p);
void png_destroy_read_struct(png_structpp p, png_infopp i, png_infopp e);
void png_destroy_write_struct(png_structpp p, png_infopp i);
jmp_buf* png_shim_jmpbuf(png_structp p);
#define png_jmpbuf(p) (*png_shim_jmpbuf(p))
void png_init_io(png_structp p, FILE* fp);
void png_set_sig_bytes(png_structp p, int n);
void png_read_info(png_structp p, png_infop i);
png_byte png_get_bit_depth(png_structp p, png_infop i);
png_byte png_get_color_type(png_structp p, png_infop i);
png_byte png_get_channels(png_structp p, png_infop i);
png_uint_32 png_get_image_width(png_structp p, png_infop i);
png_uint_32 png_get_image_height(png_structp p, png_infop i);
void png_set_expand(png_structp p);
void png_set_packing(png_structp p);
void png_set_gray_to_rgb(png_structp p);
void png_read_update_info(png_structp p, png_infop i);
void png_read_row(png_structp p, png_bytep row, png_bytep disp);
void png_read_end(png_structp p, png_infop i);
void png_set_IHDR(png_structp p, png_infop i, png_uint_32 w, png_uint_32 h, int bd, int ct, int il, int cm, int fm);
void png_write_info(png_structp p, png_infop i);
void png_write_row(png_structp p, png_const_bytep row);
void png_write_end(png_structp p, png_infop i);
#ifdef __cplusplus
}
#endif
#endif
