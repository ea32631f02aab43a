/* Stub definitions for oracle/shim/png.h (test infrastructure only). */
#include "png.h"
static jmp_buf ps_png_shim_buf;
jmp_buf* ps_png_shim_jmpbuf(png_structp p) { (void)p; return &ps_png_shim_buf; }
png_structp png_create_write_struct(const char* a, void* b, void* c, void* d) { (void)a; (void)b; (void)c; (void)d; return 0; }
png_structp png_create_read_struct(const char* a, void* b, void* c, void* d) { (void)a; (void)b; (void)c; (void)d; return 0; }
png_infop png_create_info_struct(png_structp p) { (void)p; return 0; }
void png_destroy_write_struct(png_structpp a, png_infopp b) { (void)a; (void)b; }
void png_destroy_read_struct(png_structpp a, png_infopp b, png_infopp c) { (void)a; (void)b; (void)c; }
void png_init_io(png_structp a, FILE* b) { (void)a; (void)b; }
void png_set_IHDR(png_structp a, png_infop b, png_uint_32 c, png_uint_32 d, int e, int f, int g, int h, int i) { (void)a; (void)b; (void)c; (void)d; (void)e; (void)f; (void)g; (void)h; (void)i; }
void png_write_info(png_structp a, png_infop b) { (void)a; (void)b; }
void png_write_row(png_structp a, png_bytep b) { (void)a; (void)b; }
void png_write_end(png_structp a, png_infop b) { (void)a; (void)b; }
void png_read_info(png_structp a, png_infop b) { (void)a; (void)b; }
void png_set_expand(png_structp a) { (void)a; }
void png_set_strip_16(png_structp a) { (void)a; }
void png_set_strip_alpha(png_structp a) { (void)a; }
void png_set_palette_to_rgb(png_structp a) { (void)a; }
void png_set_gray_to_rgb(png_structp a) { (void)a; }
int png_get_color_type(png_structp a, png_infop b) { (void)a; (void)b; return 0; }
void png_read_update_info(png_structp a, png_infop b) { (void)a; (void)b; }
png_uint_32 png_get_image_width(png_structp a, png_infop b) { (void)a; (void)b; return 0; }
png_uint_32 png_get_image_height(png_structp a, png_infop b) { (void)a; (void)b; return 0; }
void png_read_row(png_structp a, png_bytep b, png_bytep c) { (void)a; (void)b; (void)c; }
void png_read_end(png_structp a, png_infop b) { (void)a; (void)b; }
