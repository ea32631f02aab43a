/* Declaration-only stand-in for libpng (absent from this image) so that the
 * reference's scene_io.cpp compiles out of tree. Every png_create_* returns
 * NULL, so the reference's own error path throws IoError for PNG I/O; nothing
 * on the render path touches PNG. Test infrastructure only. */
#ifndef PS_ORACLE_PNG_SHIM_H
#define PS_ORACLE_PNG_SHIM_H
#include <setjmp.h>
#include <stdio.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef struct png_struct_def png_struct;
typedef png_struct* png_structp;
typedef struct png_info_def png_info;
typedef png_info* png_infop;
typedef png_infop* png_infopp;
typedef png_structp* png_structpp;
typedef unsigned char* png_bytep;
typedef unsigned int png_uint_32;
#define PNG_LIBPNG_VER_STRING "0.0.0-shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
jmp_buf* ps_png_shim_jmpbuf(png_structp);
#define png_jmpbuf(p) (*ps_png_shim_jmpbuf(p))
png_structp png_create_write_struct(const char*, void*, void*, void*);
png_structp png_create_read_struct(const char*, void*, void*, void*);
png_infop png_create_info_struct(png_structp);
void png_destroy_write_struct(png_structpp, png_infopp);
void png_destroy_read_struct(png_structpp, png_infopp, png_infopp);
void png_init_io(png_structp, FILE*);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_write_info(png_structp, png_infop);
void png_write_row(png_structp, png_bytep);
void png_write_end(png_structp, png_infop);
void png_read_info(png_structp, png_infop);
void png_set_expand(png_structp);
void png_set_strip_16(png_structp);
void png_set_strip_alpha(png_structp);
void png_set_palette_to_rgb(png_structp);
void png_set_gray_to_rgb(png_structp);
int png_get_color_type(png_structp, png_infop);
void png_read_update_info(png_structp, png_infop);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
void png_read_row(png_structp, png_bytep, png_bytep);
void png_read_end(png_structp, png_infop);
#ifdef __cplusplus
}
#endif
#endif
